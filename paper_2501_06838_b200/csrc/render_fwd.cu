// render_fwd.cu -- K4: forward render (Eq. 4 / Alg. 1).
//
//   I[y][x][:] = sum over records i with x0_i <= x <= x1_i, y0_i <= y <= y1_i of
//                c'_i * 2^(q_i(x,y)),   q = -(w^2 + v^2),  w = a1 dx + b1 dy,  v = c1 dy,
//                dx = (x - ax_i)/s - dl_x,  dy = (y - ay_i)/s - dl_y   (= x/s - mu_x, y/s - mu_y)
//
// CTA = one FTILE_W x FTILE_H (32 x 16) HR tile. Every warp covers the whole tile -- lane l
// owns the 2 x 8 block at columns Tx0 + 8 (l & 3) .. + 7 and rows Ty0 + 2 (l >> 2) + {0, 1} --
// for its own share of the tile's Gaussians; the partial images are summed in warp order.
//   * candidates: the tile's contiguous cell-row spans (binning.cu), walked in batches of 32 and
//     filtered from the 16-B rect stream: keep if the support rect (R21) meets the tile, "full"
//     if the window rect covers all 32 columns and 16 rows (no x mask, no y test: pixels beyond
//     the support evaluate to exactly 0 by themselves); otherwise the masked path.
//   * default (k_render_fwd2, GSR_FWD_V2=1): warp-autonomous -- each warp filters batches
//     i = warp (mod 4) and copies its kept 64-B records with per-lane cp.async into its own
//     double buffer, evaluating one buffer while the other fills.
//     Alternative (k_render_fwd, GSR_FWD_V2=0): 4 consumer warps + 1 producer warp that filters
//     and gathers runs of kept records by TMA bulk copies (cp.async.bulk, mbarrier complete_tx)
//     into a FWD_STAGES-deep ring (full / empty mbarriers per stage).
//   * per Gaussian, three paths (warp-uniform): exponential recurrence along rows (full, D <= 1:
//     2 ex2 per 4 pairs), direct (full, D > 1), masked (window edge in the tile). Direct path per
//     lane: kx = x - ax (exact small integers), w = (a1/s) kx + (b1 dy - a1 dl_x), q = -w^2 - v^2
//     (the y test folds into -v^2 -> -inf), 2^q on the SFU (ex2.approx.ftz -> MUFU.EX2),
//     colour += c' 2^q (3 FFMA2, register pairs = the lane's two rows of a column).
//   * two-level sums: per-buffer partials in registers, folded into per-warp totals in shared
//     memory.
//   * two tile configurations (gsr_internal.cuh): 2 x 8 px per lane / 32 x 16 tiles, or for
//     narrow windows 1 x 4 px per lane / 16 x 8 tiles (fewer masked evaluations).
//   * split-K for small problems: KS CTAs of a cluster share a tile, take interleaved batches,
//     and reduce their totals through DSMEM in cluster-rank order (deterministic, no atomics).
#include <atomic>
#include <mutex>

#include "gsr_internal.cuh"

#ifndef GSR_FWD_V2
#define GSR_FWD_V2 1
#endif

namespace gsr {

namespace {

struct FwdProducer {
    int cy, cy_hi, row_stride, row0, cx_lo, cx_hi, cur, end;
    const int* cs;
    __device__ int raw_next(int* start) {
        while (cur >= end) {
            if (++cy > cy_hi) return 0;
            int row = row0 + cy * row_stride;
            cur = cs[row + cx_lo];
            end = cs[row + cx_hi + 1];
        }
        int n = min(32, end - cur);
        *start = cur;
        cur += n;
        return n;
    }
    __device__ int next(int* start, int skip) {   // drop `skip` chunks, then take one
        for (int k = 0; k < skip; ++k)
            if (raw_next(start) == 0) return 0;
        return raw_next(start);
    }
};

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
                 ::: "memory");
}
__device__ __forceinline__ float2 ld_dsmem_f2(const float2* local_addr, uint32_t rank) {
    uint32_t a = smem_u32(local_addr), ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    float2 v;
    asm volatile("ld.shared::cluster.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(ra)
                 : "memory");
    return v;
}

__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }

// Column halves (GSR_FWD_HALVES, large configuration): lane l owns columns 4 (l & 3) + t and
// 16 + 4 (l & 3) + t (t = 0..3) of its two rows, so anchor h = 0 of every lane lies in the
// tile's left 16 columns and h = 1 in the right 16. A Gaussian whose support rect misses one
// half skips that anchor warp-uniformly (flag bits from the filter): at C5 about a third of the
// lane-pairs outside the supports of partly covered tiles are never evaluated.
#ifndef GSR_FWD_PACC
#define GSR_FWD_PACC 1
#endif
#ifndef GSR_FWD_HALVES
#define GSR_FWD_HALVES 1
#endif
template <int STRIP>
__device__ __forceinline__ constexpr bool use_halves() { return GSR_FWD_HALVES && STRIP == 8; }
template <int STRIP>
__device__ __forceinline__ constexpr int colx(int j) {   // tile column of the lane's slot j
    return use_halves<STRIP>() ? (j & 3) + 16 * (j >> 2) : j;
}
template <int STRIP>
__device__ __forceinline__ int lane_x0(int lane) {
    return use_halves<STRIP>() ? 4 * (lane & 3) : STRIP * (lane & 3);
}

template <class CFG>
struct FwdSmem {
    static constexpr int NACC = CFG::ROWS * (CFG::STRIP / 2) * 3;   // float2 accumulators/thread
    float4 rec[FWD_STAGES][FWD_CHUNK * REC_F4];   // kept records only (gathered by TMA)
    float2 tot[FWD_CWARPS][NACC][32];        // per-warp totals (second accumulation level)
    uint8_t full[FWD_STAGES][FWD_CHUNK];     // 1: the window rect covers the tile (no masks)
    uint64_t full_bar[FWD_STAGES];           // stage closed by the producer + its bytes landed
    uint64_t empty_bar[FWD_STAGES];          // consumer warps done with the stage
    int kept[FWD_STAGES];                    // records in the stage (-1 = end of the list)
};

// Transformed record (written in shared memory by the producer warp, see k_render_fwd):
//   r0 = {-ax, ay, dl_y, a1/s},  r1 = {-a1 dl_x, b1, c1, c'_r},
//   r2 = {c'_g, c'_b, window x0|x1, y0|y1}  (recurrence path: {c'_g, c'_b, G1, G2})
template <class CFG, bool FULL>
__device__ __forceinline__ void fwd_gauss(const float4 r0, const float4 r1, const float4 r2,
                                          const float2 (&xj)[CFG::STRIP / 2], float yf0,
                                          const int (&yi)[CFG::ROWS], int xl0, float invs,
                                          float2 (&acc)[FwdSmem<CFG>::NACC]) {
    constexpr int FWD_STRIP = CFG::STRIP, FWD_ROWS = CFG::ROWS;
    const float2 D2 = f2(r0.w);
    const float2 nax = f2(r0.x);
    // kx = x - ax for the lane's 8 columns: exact small integers (one FADD2 per column pair)
    float2 kx[FWD_STRIP / 2];
#pragma unroll
    for (int jp = 0; jp < FWD_STRIP / 2; ++jp) kx[jp] = __fadd2_rn(xj[jp], nax);
    bool cin[FWD_STRIP];
    if (!FULL) {
        const unsigned xs = __float_as_uint(r2.z);
        const int x0 = (int)(xs & 0xffffu), x1 = (int)(xs >> 16);
#pragma unroll
        for (int j = 0; j < FWD_STRIP; ++j) cin[j] = (xl0 + j >= x0) && (xl0 + j <= x1);
    }
    const float2 cr = f2(r1.w), cg = f2(r2.x), cb = f2(r2.y);
    float dy = fmaf(yf0 - r0.y, invs, -r0.z);
#pragma unroll
    for (int r = 0; r < FWD_ROWS; ++r) {
        if (r > 0) dy += invs;                               // consecutive rows: exact to 1 ulp(1/s)
        const float v = r1.z * dy;                           // c1 dy
        float u = -(v * v);
        if (!FULL) {                                         // lane's row outside [y0, y1]
            const unsigned ys = __float_as_uint(r2.w);
            const int y0 = (int)(ys & 0xffffu), y1 = (int)(ys >> 16);
            u = (yi[r] >= y0 && yi[r] <= y1) ? u : -INFINITY;
        }
        const float tau = fmaf(r1.y, dy, r1.x);              // b1 dy - a1 dl_x
        const float2 T2 = f2(tau), U2 = f2(u);
#pragma unroll
        for (int jp = 0; jp < FWD_STRIP / 2; ++jp) {
            float2 w = __ffma2_rn(D2, kx[jp], T2);
            float2 q = __ffma2_rn(make_float2(-w.x, -w.y), w, U2);
            if (!FULL) {
                q.x = cin[2 * jp] ? q.x : -INFINITY;
                q.y = cin[2 * jp + 1] ? q.y : -INFINITY;
            }
            const float2 e = make_float2(ex2_approx(q.x), ex2_approx(q.y));
            const int a = (r * (FWD_STRIP / 2) + jp) * 3;
            acc[a + 0] = __ffma2_rn(cr, e, acc[a + 0]);
            acc[a + 1] = __ffma2_rn(cg, e, acc[a + 1]);
            acc[a + 2] = __ffma2_rn(cb, e, acc[a + 2]);
        }
    }
}

// Two-row lane block (FwdCfgLarge): accumulators pair the lane's two rows of one column,
// acc[3 j + k] = (row 0, row 1) of column j, channel k. Three per-Gaussian variants:
//   MODE 0  masked:  per column, w = D kx + tau, q = -w^2 + u (x / y masks -> -inf), 2^q
//   MODE 1  full, direct: the same without masks
//   MODE 2  full, exponential recurrence (producer-flagged when D = a1/s <= FWD_REC_DMAX):
//           along a row w(kx + t) = w_a + t D, so
//             2^q(kx_a + t) = 2^q_a * B^t * G_t,  B = 2^(-2 D w_a),  G_t = 2^(-D^2 t^2),
//           evaluated at anchors j = 0, 4 (t = 1..3 from products): 2 ex2 per 4 pairs instead
//           of 4, the FMA-pipe work unchanged (w, q, -2Dw, 3 B products, 3 G products per
//           anchor vs w, q per pair). G_t come from the producer. The exponent -2 D w_a is
//           clamped to <= 40: with D <= 1 a clamped anchor has |w_a| > 20, so 2^q_a = 0 and all
//           four values are exactly 0 (B^3 <= 2^120 stays finite, no 0 * inf); an anchor whose
//           2^q_a flushes to zero (q_a < -126) has q(kx_a + 3) < -67 (|w_a| > 11.2, D <= 1),
//           i.e. only values below 2^-67 are lost; products never overflow (q <= 0 and
//           D^2 t^2 <= 9). Error: the exponent of B^t carries t * 2 D |w_a| * 2^-24 relative.
template <int MODE, int STRIP, int HSEL = 3>
__device__ __forceinline__ void fwd_gauss_r2h(const float4 r0, const float4 r1, const float4 r2,
                                              float g3, float xlf, float2 yrow, const int (&yi)[2],
                                              int xl0, float invs, float2 (&acc)[3 * STRIP]) {
    constexpr int hmask = HSEL;
    const float D = r0.w;
    const float2 D2 = f2(D);
    const float kx0 = xlf + r0.x;                           // x - ax of column 0 (exact)
    // both rows at once: dy = (y - ay)/s - dl_y ((y - ay) exact), v = c1 dy, u = -v^2,
    // tau = b1 dy - a1 dl_x
    const float2 dy = __ffma2_rn(__fadd2_rn(yrow, f2(-r0.y)), f2(invs), f2(-r0.z));
    const float2 v = __fmul2_rn(dy, f2(r1.z));
    float2 U = __fmul2_rn(make_float2(-v.x, -v.y), v);
    if (MODE == 0) {                                        // lane rows outside [y0, y1]
        const unsigned ys = __float_as_uint(r2.w);
        const int y0 = (int)(ys & 0xffffu), y1 = (int)(ys >> 16);
        U.x = (yi[0] >= y0 && yi[0] <= y1) ? U.x : -INFINITY;
        U.y = (yi[1] >= y0 && yi[1] <= y1) ? U.y : -INFINITY;
    }
    const float2 T = __ffma2_rn(f2(r1.y), dy, f2(r1.x));   // b1 dy - a1 dl_x
    const float2 cr = f2(r1.w), cg = f2(r2.x), cb = f2(r2.y);
    auto accum = [&](int j, float2 e) {
        acc[3 * j + 0] = __ffma2_rn(cr, e, acc[3 * j + 0]);
        acc[3 * j + 1] = __ffma2_rn(cg, e, acc[3 * j + 1]);
        acc[3 * j + 2] = __ffma2_rn(cb, e, acc[3 * j + 2]);
    };
    if (MODE == 2) {
        const float2 G1 = f2(r2.z), G2 = f2(r2.w), G3 = f2(g3), M2D = f2(-2.f * D);
#pragma unroll
        for (int h = 0; h < STRIP / 4; ++h) {
            if (use_halves<STRIP>() && !((hmask >> h) & 1)) continue;   // compile-time skip
            const float2 w = __ffma2_rn(D2, f2(kx0 + (float)colx<STRIP>(4 * h)), T);
            const float2 q = __ffma2_rn(make_float2(-w.x, -w.y), w, U);
            float2 b = __fmul2_rn(w, M2D);
            b.x = fminf(b.x, 40.f);
            b.y = fminf(b.y, 40.f);
            const float2 A = make_float2(ex2_approx(q.x), ex2_approx(q.y));
            const float2 B = make_float2(ex2_approx(b.x), ex2_approx(b.y));
            const float2 AB1 = __fmul2_rn(A, B);
            const float2 AB2 = __fmul2_rn(AB1, B);
            const float2 AB3 = __fmul2_rn(AB2, B);
            accum(4 * h + 0, A);
            accum(4 * h + 1, __fmul2_rn(AB1, G1));
            accum(4 * h + 2, __fmul2_rn(AB2, G2));
            accum(4 * h + 3, __fmul2_rn(AB3, G3));
        }
    } else {
        unsigned xs = 0;
        int x0 = 0, x1 = 0;
        if (MODE == 0) {
            xs = __float_as_uint(r2.z);
            x0 = (int)(xs & 0xffffu);
            x1 = (int)(xs >> 16);
        }
#pragma unroll
        for (int j = 0; j < STRIP; ++j) {
            if (use_halves<STRIP>() && !((hmask >> (j >> 2)) & 1)) continue;
            const int cj = colx<STRIP>(j);
            const float2 w = __ffma2_rn(D2, f2(kx0 + (float)cj), T);
            float2 q = __ffma2_rn(make_float2(-w.x, -w.y), w, U);
            if (MODE == 0 && !(xl0 + cj >= x0 && xl0 + cj <= x1)) q = f2(-INFINITY);
            accum(j, make_float2(ex2_approx(q.x), ex2_approx(q.y)));
        }
    }
}

// hmask (column halves the support meets, GSR_FWD_HALVES): one of three compile-time variants,
// so the evaluated anchors stay one fully unrolled, interleavable block
template <int MODE, int STRIP>
__device__ __forceinline__ void fwd_gauss_r2(const float4 r0, const float4 r1, const float4 r2,
                                             float g3, float xlf, float2 yrow, const int (&yi)[2],
                                             int xl0, float invs, float2 (&acc)[3 * STRIP],
                                             int hmask = 3) {
    if (use_halves<STRIP>() && hmask == 1)
        fwd_gauss_r2h<MODE, STRIP, 1>(r0, r1, r2, g3, xlf, yrow, yi, xl0, invs, acc);
    else if (use_halves<STRIP>() && hmask == 2)
        fwd_gauss_r2h<MODE, STRIP, 2>(r0, r1, r2, g3, xlf, yrow, yi, xl0, invs, acc);
    else
        fwd_gauss_r2h<MODE, STRIP, 3>(r0, r1, r2, g3, xlf, yrow, yi, xl0, invs, acc);
}

// Sum the per-warp partial images in warp order (deterministic) into tot[0], reduce split-K
// cluster CTAs through DSMEM in rank order, store the tile (and the fused L1 loss).
template <int KS, bool LOSS, class CFG>
__device__ __forceinline__ void fwd_epilogue(float2 (*tot)[FwdSmem<CFG>::NACC][32],
                                             const DevImg& im, int Tx0, int Ty0, int warp,
                                             int lane, int krank, float* __restrict__ out,
                                             const float* __restrict__ gt,
                                             double* __restrict__ loss_acc) {
    constexpr int FWD_STRIP = CFG::STRIP, FWD_ROWS = CFG::ROWS, NACC = FwdSmem<CFG>::NACC;
    struct { float2 (*tot)[NACC][32]; } sm = {tot};
    __syncthreads();
    if (warp == 0) {
#pragma unroll 4
        for (int a = 0; a < NACC; ++a) {
            float2 v = sm.tot[0][a][lane];
            for (int q = 1; q < FWD_CWARPS; ++q) v = __fadd2_rn(v, sm.tot[q][a][lane]);
            sm.tot[0][a][lane] = v;
        }
    }
    if (KS > 1) {
        cluster_sync_all();                    // every CTA's tile sum is final
        if (krank == 0 && warp == 0) {
            for (int a = 0; a < NACC; ++a) {
                float2 v = make_float2(0.f, 0.f);
                for (int q = 0; q < KS; ++q) v = __fadd2_rn(v, ld_dsmem_f2(&sm.tot[0][a][lane], q));
                sm.tot[0][a][lane] = v;        // only this thread reads its own slot afterwards
            }
        }
        cluster_sync_all();                    // keep every CTA's smem alive until read
        if (krank != 0) return;
    }
    if (warp != 0) return;

    const int xl0 = Tx0 + lane_x0<FWD_STRIP>(lane);
    const int yl0 = Ty0 + FWD_ROWS * (lane >> 2);
    float l1 = 0.f;     // fused L1 loss (NEXT-1): sum |I - I_gt| over the stored elements
    auto store = [&](int y, int x, float R, float G, float B) {
        if (y >= im.row_end || x >= im.Ws) return;
        if (!LOSS && im.io != 0) {     // NEXT-4 image formats (bf16 and/or planar CHW)
            img_store(out, im, img_index(im, y, x, 0), R);
            img_store(out, im, img_index(im, y, x, 1), G);
            img_store(out, im, img_index(im, y, x, 2), B);
            return;
        }
        const long long off = im.out_off + ((long long)(y - im.row_begin) * im.Ws + x) * 3;
        out[off] = R; out[off + 1] = G; out[off + 2] = B;
        if (LOSS) l1 += fabsf(R - gt[off]) + fabsf(G - gt[off + 1]) + fabsf(B - gt[off + 2]);
    };
    if constexpr (FWD_ROWS == 2) {     // acc pairs = (row 0, row 1) of one column
#pragma unroll
        for (int j = 0; j < FWD_STRIP; ++j) {
            const float2 R = sm.tot[0][3 * j][lane], G = sm.tot[0][3 * j + 1][lane],
                         B = sm.tot[0][3 * j + 2][lane];
            store(yl0, xl0 + colx<FWD_STRIP>(j), R.x, G.x, B.x);
            store(yl0 + 1, xl0 + colx<FWD_STRIP>(j), R.y, G.y, B.y);
        }
    } else {                           // acc pairs = two adjacent columns of one row
#pragma unroll
        for (int r = 0; r < FWD_ROWS; ++r) {
#pragma unroll
            for (int jp = 0; jp < FWD_STRIP / 2; ++jp) {
                const int a = (r * (FWD_STRIP / 2) + jp) * 3;
                const float2 R = sm.tot[0][a][lane], G = sm.tot[0][a + 1][lane],
                             B = sm.tot[0][a + 2][lane];
                store(yl0 + r, xl0 + 2 * jp, R.x, G.x, B.x);
                store(yl0 + r, xl0 + 2 * jp + 1, R.y, G.y, B.y);
            }
        }
    }
    if (LOSS) {
        double d = (double)l1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        if (lane == 0) atomicAdd(loss_acc, d);
    }
}

template <int KS, bool LOSS, class CFG>
__global__ void __launch_bounds__(FWD_THREADS) k_render_fwd(const ImgTable tab,
                                                            const float4* __restrict__ rec,
                                                            const int4* __restrict__ rects,
                                                            const int* __restrict__ cell_start,
                                                            const int* __restrict__ ext,
                                                            float* __restrict__ out,
                                                            const float* __restrict__ gt,
                                                            double* __restrict__ loss_acc) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    FwdSmem<CFG>& sm = *reinterpret_cast<FwdSmem<CFG>*>(smem_raw);
    constexpr int FTILE_W = CFG::TW, FTILE_H = CFG::TH, FWD_STRIP = CFG::STRIP,
                  FWD_ROWS = CFG::ROWS, NACC = FwdSmem<CFG>::NACC;

    const int tile = blockIdx.x / KS;
    const int krank = KS > 1 ? (int)cluster_rank() : 0;
    const int kimg = find_image_by_ftile(tab, tile);
    const DevImg& im = tab.img[kimg];
    const int t = tile - im.ftile_base;
    const int Tx0 = (t % im.fntx) * FTILE_W;
    const int Ty0 = im.row_begin + (t / im.fntx) * FTILE_H;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < FWD_STAGES; ++s) {
            mbar_init(&sm.full_bar[s], 1);
            mbar_init(&sm.empty_bar[s], FWD_CWARPS);
        }
        fence_barrier_init();
    }
    for (int i = threadIdx.x; i < FWD_CWARPS * NACC * 32; i += FWD_THREADS)
        (&sm.tot[0][0][0])[i] = make_float2(0.f, 0.f);
    __syncthreads();

    const int fx0 = Tx0, fx1 = min(Tx0 + FTILE_W - 1, im.Ws - 1);   // tile footprint
    const int fy0 = Ty0, fy1 = min(Ty0 + FTILE_H - 1, im.row_end - 1);
    const float invs = im.invsy;     // rows: dy = (y - ay)/sy - dl_y

    if (warp == FWD_CWARPS) {
        // ---------------- producer warp --------------------------------------------------------
        // Walks the tile's candidate spans in batches of 32 and filters them from the 16-B rect
        // stream (support rect meets the tile? window rect covers it?), FOUR batches of loads in
        // flight; each lane whose candidate is kept issues a 64-B TMA bulk copy of its record
        // into the next free slot of the current stage (mbarrier expect_tx per copy), so the
        // stages hold kept records only. A stage is closed (one arrive on its full barrier) when
        // it cannot take another batch; the consumers see it once all its bytes have landed.
        FwdProducer prod;
        prod.cs = cell_start;
        prod.row0 = im.cell_base;
        prod.row_stride = im.ncx;
        prod.cx_lo = (Tx0 - query_ext(ext, kimg, 0) + 1 + im.offx) / CELL;
        prod.cx_hi = min(im.ncx - 1, (fx1 + im.offx) / CELL);
        prod.cy = (Ty0 - im.row_begin - query_ext(ext, kimg, 1) + 1 + im.offy) / CELL - 1;
        prod.cy_hi = min(im.ncy - 1, (fy1 - im.row_begin + im.offy) / CELL);
        prod.cur = prod.end = 0;
        const unsigned lt = (1u << lane) - 1u;
        const bool live = fy0 <= fy1;
        int nb[4], sb[4];                         // batch descriptors (warp-uniform)
        int4 rb[4];                               // this lane's rect in each batch
        int first = 1;
        auto fetch = [&](int j) {
            nb[j] = live ? prod.next(&sb[j], first ? krank : KS - 1) : 0;
            first = 0;
            rb[j] = make_int4(0, 0, 0, 0);
            if (lane < nb[j]) rb[j] = __ldg(rects + sb[j] + lane);
        };
        fetch(0); fetch(1); fetch(2); fetch(3);
        int k = 0, kept = 0;
        bool done = false;
        // the batch ring is walked with static indices (unrolled by 4): batch j is filtered, then
        // its slot is refilled with the batch four ahead
        while (!done) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if (done) break;
                const int s = k % FWD_STAGES;
                const bool end = nb[j] == 0;
                if (!end) {
                    bool keep = false, full = false;
                    if (lane < nb[j]) {
                        const unsigned sxs = (unsigned)rb[j].x, sys = (unsigned)rb[j].y;
                        const int sx0 = (int)(sxs & 0xffffu), sx1 = (int)(sxs >> 16);
                        const int sy0 = (int)(sys & 0xffffu), sy1 = (int)(sys >> 16);
                        keep = !(sx1 < fx0 || sx0 > fx1 || sy1 < fy0 || sy0 > fy1);
                        const unsigned xs = (unsigned)rb[j].z, ys = (unsigned)rb[j].w;
                        const int x0 = (int)(xs & 0xffffu), x1 = (int)(xs >> 16);
                        const int y0 = (int)(ys & 0xffffu), y1 = (int)(ys >> 16);
                        full = x0 <= fx0 && x1 >= fx1 && y0 <= fy0 && y1 >= fy0 + FTILE_H - 1;
                    }
                    const unsigned m = __ballot_sync(0xffffffffu, keep);
                    if (keep) {
                        const int slot = kept + __popc(m & lt);
                        sm.full[s][slot] = full ? 1 : 0;
                        // one bulk copy per run of consecutive kept candidates (contiguous in
                        // the source and in the stage): the copies take warp-uniform operands,
                        // so every copy costs a serialised issue round
                        if (lane == 0 || !((m >> (lane - 1)) & 1u)) {
                            const int run = __ffsll(~(unsigned long long)(m >> lane)) - 1;
                            const uint32_t bytes = (uint32_t)run * (16u * REC_F4);
                            mbar_expect_tx(&sm.full_bar[s], bytes);
                            tma_bulk_g2s(&sm.rec[s][REC_F4 * slot],
                                         rec + (long long)REC_F4 * (sb[j] + lane), bytes,
                                         &sm.full_bar[s]);
                        }
                    }
                    kept += __popc(m);
                    fetch(j);                     // the batch four ahead
                }
                if (kept > FWD_CHUNK - 32 || (end && kept > 0)) {
                    // close stage s
                    if (lane == 0) sm.kept[s] = kept;
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&sm.full_bar[s]);
                    ++k;
                    kept = 0;
                    if (k >= FWD_STAGES)      // wait until the consumers released the next stage
                        mbar_wait(&sm.empty_bar[k % FWD_STAGES],
                                  (uint32_t)(((k / FWD_STAGES) - 1) & 1));
                }
                if (end) {
                    const int s2 = k % FWD_STAGES;
                    if (lane == 0) {
                        sm.kept[s2] = -1;
                        mbar_arrive(&sm.full_bar[s2]);
                    }
                    done = true;
                }
            }
        }
    } else {
        // ---------------- consumer warps ------------------------------------------------------
        const int xl0 = Tx0 + lane_x0<FWD_STRIP>(lane);
        const int yl0 = Ty0 + FWD_ROWS * (lane >> 2);
        float2 xj[FWD_STRIP / 2];
#pragma unroll
        for (int jp = 0; jp < FWD_STRIP / 2; ++jp)
            xj[jp] = make_float2((float)(xl0 + 2 * jp), (float)(xl0 + 2 * jp + 1));
        const float xlf = (float)xl0;
        const float2 yrow = make_float2((float)yl0, (float)(yl0 + 1));
        int yi[FWD_ROWS];
#pragma unroll
        for (int r = 0; r < FWD_ROWS; ++r) yi[r] = yl0 + r;
        const float yf0 = (float)yl0;

        for (int k = 0;; ++k) {
            const int s = k % FWD_STAGES;
            mbar_wait(&sm.full_bar[s], (uint32_t)((k / FWD_STAGES) & 1));
            const int nk = sm.kept[s];
            if (nk < 0) break;
            float2 acc[NACC];
#pragma unroll
            for (int a = 0; a < NACC; ++a) acc[a] = make_float2(0.f, 0.f);
            const float4* sr = &sm.rec[s][0];
            for (int g = warp; g < nk; g += FWD_CWARPS) {
                const float4 r0 = sr[REC_F4 * g], r1 = sr[REC_F4 * g + 1],
                             r2 = sr[REC_F4 * g + 2];
                const bool full = sm.full[s][g] != 0;
                if constexpr (FWD_ROWS == 2) {
                    if (full) {
                        const float4 r3 = sr[REC_F4 * g + 3];
                        if (r3.w != 0.f)
                            fwd_gauss_r2<2, FWD_STRIP>(r0, r1, make_float4(r2.x, r2.y, r3.x, r3.y), r3.z, xlf,
                                            yrow, yi, xl0, invs, acc);
                        else
                            fwd_gauss_r2<1, FWD_STRIP>(r0, r1, r2, 0.f, xlf, yrow, yi, xl0, invs, acc);
                    } else {
                        fwd_gauss_r2<0, FWD_STRIP>(r0, r1, r2, 0.f, xlf, yrow, yi, xl0, invs, acc);
                    }
                } else {
                    if (full)
                        fwd_gauss<CFG, true>(r0, r1, r2, xj, yf0, yi, xl0, invs, acc);
                    else
                        fwd_gauss<CFG, false>(r0, r1, r2, xj, yf0, yi, xl0, invs, acc);
                }
            }
            // fold the stage partials into the per-warp totals (second accumulation level)
#pragma unroll
            for (int a = 0; a < NACC; ++a)
                sm.tot[warp][a][lane] = __fadd2_rn(sm.tot[warp][a][lane], acc[a]);
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.empty_bar[s]);
        }
    }

    fwd_epilogue<KS, LOSS, CFG>(sm.tot, im, Tx0, Ty0, warp, lane, krank, out, gt, loss_acc);
}

// ------------------------------------------------------------------------------------------
// K4, warp-autonomous variant (no producer warp): every warp filters its own share of the
// tile's candidate batches (batch i of the tile goes to warp i mod 4, and to cluster CTA
// (i / 4) mod KS) from the rect stream, copies its kept records into its own double buffer in
// shared memory with per-lane cp.async (16-B, L2 -> smem, no uniform-operand serialisation),
// and evaluates buffer k while the copies of buffer k + 1 are in flight. All warps still cover
// the whole tile; each sums its own Gaussians, and the warp images are added in warp order.
#ifndef GSR_FWD_PAIR
#define GSR_FWD_PAIR 0            // 1: recurrence-path Gaussians two at a time (measured 1% slower)
#endif
#ifndef GSR_FWD_MINB
#define GSR_FWD_MINB 4            // CTAs per SM the register allocation must allow
#endif
#ifndef GSR_FWD_BUF
#define GSR_FWD_BUF 48
#endif
constexpr int FWD_BUF = GSR_FWD_BUF;              // records per warp buffer (> 32)
constexpr int FWD2_THREADS = FWD_CWARPS * 32;

template <class CFG>
struct FwdSmem2 {
    float4 rec[FWD_CWARPS][2][FWD_BUF * REC_F4];
    uint8_t full[FWD_CWARPS][2][FWD_BUF];
    float2 tot[FWD_CWARPS][FwdSmem<CFG>::NACC][32];
};


template <int KS, bool LOSS, class CFG>
__global__ void __launch_bounds__(FWD2_THREADS, GSR_FWD_MINB) k_render_fwd2(const ImgTable tab,
                                                              const float4* __restrict__ rec,
                                                              const int4* __restrict__ rects,
                                                              const int* __restrict__ cell_start,
                                                              const int* __restrict__ ext,
                                                              float* __restrict__ out,
                                                              const float* __restrict__ gt,
                                                              double* __restrict__ loss_acc) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    FwdSmem2<CFG>& sm = *reinterpret_cast<FwdSmem2<CFG>*>(smem_raw);
    constexpr int FTILE_W = CFG::TW, FTILE_H = CFG::TH, FWD_STRIP = CFG::STRIP,
                  FWD_ROWS = CFG::ROWS, NACC = FwdSmem<CFG>::NACC;

    const int tile = blockIdx.x / KS;
    const int krank = KS > 1 ? (int)cluster_rank() : 0;
    const int kimg = find_image_by_ftile(tab, tile);
    const DevImg& im = tab.img[kimg];
    const int t = tile - im.ftile_base;
    const int Tx0 = (t % im.fntx) * FTILE_W;
    const int Ty0 = im.row_begin + (t / im.fntx) * FTILE_H;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    for (int a = 0; a < NACC; ++a) sm.tot[warp][a][lane] = make_float2(0.f, 0.f);

    const int fx0 = Tx0, fx1 = min(Tx0 + FTILE_W - 1, im.Ws - 1);   // tile footprint
    const int fy0 = Ty0, fy1 = min(Ty0 + FTILE_H - 1, im.row_end - 1);
    const float invs = im.invsy;     // rows: dy = (y - ay)/sy - dl_y

    // lane geometry (every warp covers the whole tile)
    const int xl0 = Tx0 + lane_x0<FWD_STRIP>(lane);
    const int yl0 = Ty0 + FWD_ROWS * (lane >> 2);
    float2 xj[FWD_STRIP / 2];
#pragma unroll
    for (int jp = 0; jp < FWD_STRIP / 2; ++jp)
        xj[jp] = make_float2((float)(xl0 + 2 * jp), (float)(xl0 + 2 * jp + 1));
    const float xlf = (float)xl0;
    const float2 yrow = make_float2((float)yl0, (float)(yl0 + 1));
    int yi[FWD_ROWS];
#pragma unroll
    for (int r = 0; r < FWD_ROWS; ++r) yi[r] = yl0 + r;
    const float yf0 = (float)yl0;

    FwdProducer prod;
    prod.cs = cell_start;
    prod.row0 = im.cell_base;
    prod.row_stride = im.ncx;
    prod.cx_lo = (Tx0 - query_ext(ext, kimg, 0) + 1 + im.offx) / CELL;
    prod.cx_hi = min(im.ncx - 1, (fx1 + im.offx) / CELL);
    prod.cy = (Ty0 - im.row_begin - query_ext(ext, kimg, 1) + 1 + im.offy) / CELL - 1;
    prod.cy_hi = min(im.ncy - 1, (fy1 - im.row_begin + im.offy) / CELL);
    prod.cur = prod.end = 0;
    const unsigned lt = (1u << lane) - 1u;
    const bool live = fy0 <= fy1;
    int nb[2], sb[2];
    int4 rb[2];
    int first = 1;
    auto fetch = [&](int j) {
        nb[j] = live ? prod.next(&sb[j], first ? krank * FWD_CWARPS + warp
                                               : KS * FWD_CWARPS - 1) : 0;
        first = 0;
        rb[j] = make_int4(0, 0, 0, 0);
        if (lane < nb[j]) rb[j] = __ldg(rects + sb[j] + lane);
    };

#if GSR_FWD_PACC
    // experiment: one register accumulator per lane for the whole tile (no per-buffer folds)
    float2 acc[NACC];
#pragma unroll
    for (int a = 0; a < NACC; ++a) acc[a] = make_float2(0.f, 0.f);
#endif
    auto process = [&](int pbuf, int pcnt) {
#if !GSR_FWD_PACC
        float2 acc[NACC];
#pragma unroll
        for (int a = 0; a < NACC; ++a) acc[a] = make_float2(0.f, 0.f);
#endif
        const float4* sr = &sm.rec[warp][pbuf][0];
        auto single = [&](int g) {
            const float4 r0 = sr[REC_F4 * g], r1 = sr[REC_F4 * g + 1], r2 = sr[REC_F4 * g + 2];
            const int fl = sm.full[warp][pbuf][g];
            const bool full = (fl & 1) != 0;
            const int hm = fl >> 1;
            if constexpr (FWD_ROWS == 2) {
                if (full) {
                    const float4 r3 = sr[REC_F4 * g + 3];
                    if (r3.w != 0.f)
                        fwd_gauss_r2<2, FWD_STRIP>(r0, r1, make_float4(r2.x, r2.y, r3.x, r3.y),
                                                   r3.z, xlf, yrow, yi, xl0, invs, acc, hm);
                    else
                        fwd_gauss_r2<1, FWD_STRIP>(r0, r1, r2, 0.f, xlf, yrow, yi, xl0, invs, acc,
                                                   hm);
                } else {
                    fwd_gauss_r2<0, FWD_STRIP>(r0, r1, r2, 0.f, xlf, yrow, yi, xl0, invs, acc,
                                               hm);
                }
            } else {
                if (full)
                    fwd_gauss<CFG, true>(r0, r1, r2, xj, yf0, yi, xl0, invs, acc);
                else
                    fwd_gauss<CFG, false>(r0, r1, r2, xj, yf0, yi, xl0, invs, acc);
            }
        };
        int g = 0;
        while (g < pcnt) {
#if GSR_FWD_PAIR
            if constexpr (FWD_ROWS == 2) {
                // two recurrence-path Gaussians in one basic block: independent chains the
                // scheduler interleaves (the kernel is latency-bound at 4 warps per SMSP)
                if (g + 1 < pcnt) {
                    const float4 a3 = sr[REC_F4 * g + 3], b3 = sr[REC_F4 * (g + 1) + 3];
                    const int fa = sm.full[warp][pbuf][g], fb = sm.full[warp][pbuf][g + 1];
                    if ((fa & 1) && (fb & 1) &&
                        a3.w != 0.f && b3.w != 0.f) {
                        const float4 a0 = sr[REC_F4 * g], a1 = sr[REC_F4 * g + 1],
                                     a2 = sr[REC_F4 * g + 2];
                        const float4 b0 = sr[REC_F4 * (g + 1)], b1 = sr[REC_F4 * (g + 1) + 1],
                                     b2 = sr[REC_F4 * (g + 1) + 2];
                        fwd_gauss_r2<2, FWD_STRIP>(a0, a1, make_float4(a2.x, a2.y, a3.x, a3.y),
                                                   a3.z, xlf, yrow, yi, xl0, invs, acc, fa >> 1);
                        fwd_gauss_r2<2, FWD_STRIP>(b0, b1, make_float4(b2.x, b2.y, b3.x, b3.y),
                                                   b3.z, xlf, yrow, yi, xl0, invs, acc, fb >> 1);
                        g += 2;
                        continue;
                    }
                }
            }
#endif
            single(g);
            ++g;
        }
#if !GSR_FWD_PACC
#pragma unroll
        for (int a = 0; a < NACC; ++a)
            sm.tot[warp][a][lane] = __fadd2_rn(sm.tot[warp][a][lane], acc[a]);
#endif
    };

    fetch(0);
    fetch(1);
    int b = 0, cnt = 0, pend = -1;
    while (true) {
        const bool end = nb[0] == 0;
        if (!end) {
            bool keep = false, full = false;
            int hb = 3;
            if (lane < nb[0]) {
                const unsigned sxs = (unsigned)rb[0].x, sys = (unsigned)rb[0].y;
                const int sx0 = (int)(sxs & 0xffffu), sx1 = (int)(sxs >> 16);
                const int sy0 = (int)(sys & 0xffffu), sy1 = (int)(sys >> 16);
                keep = !(sx1 < fx0 || sx0 > fx1 || sy1 < fy0 || sy0 > fy1);
                const unsigned xs = (unsigned)rb[0].z, ys = (unsigned)rb[0].w;
                const int x0 = (int)(xs & 0xffffu), x1 = (int)(xs >> 16);
                const int y0 = (int)(ys & 0xffffu), y1 = (int)(ys >> 16);
                full = x0 <= fx0 && x1 >= fx1 && y0 <= fy0 && y1 >= fy0 + FTILE_H - 1;
                // column halves the support meets (bit 0: left 16 columns, bit 1: right 16)
                hb = use_halves<FWD_STRIP>()
                         ? (sx0 <= fx0 + 15 ? 1 : 0) | (sx1 >= fx0 + 16 ? 2 : 0) : 3;
            }
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const int slot = cnt + __popc(m & lt);
                sm.full[warp][b][slot] = (uint8_t)((full ? 1 : 0) | (hb << 1));
                const float4* src = rec + (long long)REC_F4 * (sb[0] + lane);
                float4* dst = &sm.rec[warp][b][REC_F4 * slot];
#pragma unroll
                for (int q = 0; q < REC_F4; ++q) cp_async16(dst + q, src + q);
            }
            cnt += __popc(m);
            nb[0] = nb[1]; sb[0] = sb[1]; rb[0] = rb[1];
            fetch(1);
        }
        if (cnt > FWD_BUF - 32 || (end && cnt > 0)) {
            cp_async_commit();
            if (pend >= 0) {                  // the other buffer: its copies are older
                cp_async_wait<1>();
                __syncwarp();
                process(b ^ 1, pend);
                __syncwarp();
            }
            pend = cnt;
            b ^= 1;
            cnt = 0;
        }
        if (end) break;
    }
    if (pend >= 0) {
        cp_async_wait<0>();
        __syncwarp();
        process(b ^ 1, pend);
    }
#if GSR_FWD_PACC
#pragma unroll
    for (int a = 0; a < NACC; ++a) sm.tot[warp][a][lane] = acc[a];
#endif
    fwd_epilogue<KS, LOSS, CFG>(sm.tot, im, Tx0, Ty0, warp, lane, krank, out, gt, loss_acc);
}

// one-time function setup of an instance (also loads its code under CUDA lazy loading)
template <int KS, bool LOSS, class CFG>
cudaError_t fwd2_prepare() {
    static std::atomic<bool> attr_set{false};    // concurrent first calls just repeat the set
    if (!attr_set.load(std::memory_order_acquire)) {
        cudaError_t e = cudaFuncSetAttribute(k_render_fwd2<KS, LOSS, CFG>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)sizeof(FwdSmem2<CFG>));
        if (e != cudaSuccess) return e;
        attr_set.store(true, std::memory_order_release);
    }
    return cudaSuccess;
}

template <int KS, bool LOSS, class CFG>
cudaError_t launch_ks3_v2(const ImgTable& tab, const Workspace& ws, float* out, const float* gt,
                          double* loss_acc, cudaStream_t st) {
    const size_t smem = sizeof(FwdSmem2<CFG>);
    cudaError_t e0 = fwd2_prepare<KS, LOSS, CFG>();
    if (e0 != cudaSuccess) return e0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)tab.total_ftiles * KS);
    cfg.blockDim = dim3(FWD2_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = KS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_render_fwd2<KS, LOSS, CFG>, tab, (const float4*)ws.rec,
                              (const int4*)ws.rects, (const int*)ws.cell_start,
                              (const int*)ws.ext, out, gt, loss_acc);
}

template <int KS, bool LOSS, class CFG>
cudaError_t launch_ks3(const ImgTable& tab, const Workspace& ws, float* out, const float* gt,
                       double* loss_acc, cudaStream_t st) {
    static std::atomic<bool> attr_set{false};
    const size_t smem = sizeof(FwdSmem<CFG>);
    if (!attr_set.load(std::memory_order_acquire)) {
        cudaError_t e = cudaFuncSetAttribute(k_render_fwd<KS, LOSS, CFG>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        attr_set.store(true, std::memory_order_release);
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)tab.total_ftiles * KS);
    cfg.blockDim = dim3(FWD_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = KS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_render_fwd<KS, LOSS, CFG>, tab, (const float4*)ws.rec,
                              (const int4*)ws.rects, (const int*)ws.cell_start, (const int*)ws.ext, out, gt,
                              loss_acc);
}

template <int KS, bool LOSS>
cudaError_t launch_ks2(const ImgTable& tab, const Workspace& ws, float* out, const float* gt,
                       double* loss_acc, cudaStream_t st) {
#if GSR_FWD_V2
    return tab.fwd_small ? launch_ks3_v2<KS, LOSS, FwdCfgSmall>(tab, ws, out, gt, loss_acc, st)
                         : launch_ks3_v2<KS, LOSS, FwdCfgWide>(tab, ws, out, gt, loss_acc, st);
#else
    return tab.fwd_small ? launch_ks3<KS, LOSS, FwdCfgSmall>(tab, ws, out, gt, loss_acc, st)
                         : launch_ks3<KS, LOSS, FwdCfgWide>(tab, ws, out, gt, loss_acc, st);
#endif
}

template <int KS>
cudaError_t launch_ks(const ImgTable& tab, const Workspace& ws, float* out, const float* gt,
                      double* loss_acc, cudaStream_t st) {
    return gt ? launch_ks2<KS, true>(tab, ws, out, gt, loss_acc, st)
              : launch_ks2<KS, false>(tab, ws, out, gt, loss_acc, st);
}

// co-resident forward CTAs of a configuration (the split-K choice depends on it)
template <class CFG>
int fwd_slots() {
#if GSR_FWD_V2
    const auto k = k_render_fwd2<1, false, CFG>;
    const size_t smem = sizeof(FwdSmem2<CFG>);
    const int threads = FWD2_THREADS;
#else
    const auto k = k_render_fwd<1, false, CFG>;
    const size_t smem = sizeof(FwdSmem<CFG>);
    const int threads = FWD_THREADS;
#endif
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return resident_slots(k, threads, smem);
}

}  // namespace

cudaError_t launch_render_fwd(const ImgTable& tab, const Workspace& ws, float* out,
                              cudaStream_t st, const float* gt, double* loss_acc) {
    if (tab.total_ftiles <= 0) return cudaSuccess;
    count_launches(1);
    int h = prof_begin(1, st);
    // split-K (cluster CTAs share a tile) so that small problems fill the SMs without a mostly
    // idle last wave
#if GSR_FWD_V2
    // every instance the split choice can pick is set up (and its code loaded) on the first
    // call, so a later batch with a new split factor does not pay a module load mid-stream
    static std::once_flag prepared;
    std::call_once(prepared, [] {
        fwd2_prepare<1, false, FwdCfgSmall>(); fwd2_prepare<2, false, FwdCfgSmall>();
        fwd2_prepare<4, false, FwdCfgSmall>(); fwd2_prepare<8, false, FwdCfgSmall>();
        fwd2_prepare<1, true, FwdCfgSmall>(); fwd2_prepare<2, true, FwdCfgSmall>();
        fwd2_prepare<4, true, FwdCfgSmall>(); fwd2_prepare<8, true, FwdCfgSmall>();
        fwd2_prepare<1, false, FwdCfgWide>(); fwd2_prepare<2, false, FwdCfgWide>();
        fwd2_prepare<4, false, FwdCfgWide>(); fwd2_prepare<8, false, FwdCfgWide>();
        fwd2_prepare<1, true, FwdCfgWide>(); fwd2_prepare<2, true, FwdCfgWide>();
        fwd2_prepare<4, true, FwdCfgWide>(); fwd2_prepare<8, true, FwdCfgWide>();
    });
#endif
    static std::atomic<int> slots_small{0}, slots_wide{0};
    std::atomic<int>& sl = tab.fwd_small ? slots_small : slots_wide;
    int slots = sl.load(std::memory_order_relaxed);
    if (slots == 0) {
        slots = tab.fwd_small ? fwd_slots<FwdCfgSmall>() : fwd_slots<FwdCfgWide>();
        sl.store(slots, std::memory_order_relaxed);
    }
    const int ks = split_k_factor(tab.total_ftiles, slots);
    cudaError_t e;
    switch (ks) {
        case 8: e = launch_ks<8>(tab, ws, out, gt, loss_acc, st); break;
        case 4: e = launch_ks<4>(tab, ws, out, gt, loss_acc, st); break;
        case 2: e = launch_ks<2>(tab, ws, out, gt, loss_acc, st); break;
        default: e = launch_ks<1>(tab, ws, out, gt, loss_acc, st); break;
    }
    prof_end(h, st);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

}  // namespace gsr
