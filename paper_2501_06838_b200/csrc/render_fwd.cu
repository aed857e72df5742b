// render_fwd.cu -- K4: forward render (Eq. 4 / Alg. 1).
//
//   I[y][x][:] = sum over records i with x0_i <= x <= x1_i, y0_i <= y <= y1_i of
//                c'_i * 2^(q_i(x,y)),   q = -(w^2 + v^2),  w = a1 dx + b1 dy,  v = c1 dy,
//                dx = (x - ax_i)/s - dl_x,  dy = (y - ay_i)/s - dl_y   (= x/s - mu_x, y/s - mu_y)
//
// CTA = one FTILE_W x FTILE_H (32 x 16) HR tile, W = CFG::WARPS warps (2; 4 for the small tiles).
// Every warp covers the whole tile -- lane l owns the 2 x 8 block at columns Tx0 + 4 (l & 3) +
// {0..3, 16..19} and rows Ty0 + 2 (l >> 2) + {0, 1} -- for its own share of the tile's Gaussians;
// the partial images are summed in warp order.
//   * candidates: the tile's cell-row spans (binning.cu), each trimmed to the cells whose reach
//     meets the tile, concatenated into one stream (CandStream) and interleaved over the KS W
//     warps of the (split-K cluster of) CTA(s) at the lane level, filtered from the 16-B rect
//     stream + the record class byte: keep if the support rect (R21) meets the tile; the filter
//     also decides the Gaussian's evaluation PATH (below).
//   * staging: each lane whose candidate is kept copies its 64-B record with four 16-B cp.async
//     into the warp's own double buffer in shared memory -- the dominant path (recurrence over
//     both column halves / the unmasked small tile) from the buffer's front, every other path
//     from its back with a path byte -- and a warp evaluates one buffer while the copies of the
//     other are in flight: the front run without any per-Gaussian dispatch (the dispatch's
//     dependent compare-and-branch chain held ~25% of the stall samples), then the back.
//   * paths (warp-uniform per Gaussian): exponential recurrence along rows (window rect covers
//     the tile and D <= 1: 2 ex2 per 4 pairs), direct (covers, D > 1), masked (a window edge
//     crosses the tile); each in three column-half variants (support meets the left 16, the
//     right 16 or both columns), compile-time so the evaluated anchors stay one unrolled block.
//   * sums: one register accumulator per lane-pixel for the whole tile; at the end all warps
//     add the warp images (in warp order, deterministic) into an HWC staging tile in shared
//     memory, reduce split-K cluster CTAs through DSMEM in rank order, and store the tile with
//     coalesced 16-B (float4) stores (scalar at ragged image edges / misaligned rows).
//   * two tile configurations (gsr_internal.cuh): 2 x 8 px per lane / 32 x 16 tiles, or for
//     narrow windows 1 x 4 px per lane / 16 x 8 tiles (fewer masked evaluations); a 2 x 8 (or,
//     as a build option, 1 x 8) block skips the column half of the tile a Gaussian's support misses.
#include <atomic>
#include <mutex>

#include "gsr_internal.cuh"

#ifndef GSR_FWD_SCAN_D
#define GSR_FWD_SCAN_D 2          // candidate batches per warp in the scan pipeline (>= 2)
#endif

namespace gsr {

namespace {

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
                 ::: "memory");
}
__device__ __forceinline__ float ld_dsmem_f(const float* local_addr, uint32_t rank) {
    uint32_t a = smem_u32(local_addr), ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(ra) : "memory");
    return v;
}

// Column halves (large configuration): lane l owns columns 4 (l & 3) + t and 16 + 4 (l & 3) + t
// (t = 0..3) of its two rows, so anchor h = 0 of every lane lies in the tile's left 16 columns
// and h = 1 in the right 16. A Gaussian whose support rect misses one half skips that anchor.
template <int STRIP>
__device__ __forceinline__ constexpr bool use_halves() { return STRIP == 8; }
template <int STRIP>
__device__ __forceinline__ constexpr int colx(int j) {   // tile column of the lane's slot j
    return use_halves<STRIP>() ? (j & 3) + 16 * (j >> 2) : j;
}
template <int STRIP>
__device__ __forceinline__ int lane_x0(int lane) {
    return use_halves<STRIP>() ? 4 * (lane & 3) : STRIP * (lane & 3);
}

template <class CFG>
struct FwdAcc { static constexpr int NACC = CFG::ROWS * (CFG::STRIP / 2) * 3; };   // float2s

__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }

// 16-B shared load at a 32-bit shared-window address (volatile: stays after the cp.async wait)
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}

// Staged record (binning.cu K1b): r0 = {-ax, ay, dl_y, a1/s},  r1 = {-a1 dl_x, b1, c1, c'_r},
//   r2 = {c'_g, c'_b, window x0|x1, y0|y1}  (recurrence path: {c'_g, c'_b, G1, G2})
// Masked (FULL = false): mw = the window rect as tile masks written by the filter (bit c of
// mw.x: tile column c inside the window, bit r of mw.y: tile row r), xo / yo = the lane's
// first column / row in the tile.
template <class CFG, bool FULL, int HSEL = 3>
__device__ __forceinline__ void fwd_gauss(const float4 r0, const float4 r1, const float4 r2,
                                          uint2 mw, const float2 (&xj)[CFG::STRIP / 2],
                                          float yf0, int xo, int yo, float invs,
                                          float2 (&acc)[FwdAcc<CFG>::NACC]) {
    constexpr int FWD_STRIP = CFG::STRIP, FWD_ROWS = CFG::ROWS;
    const float2 D2 = f2(r0.w);
    const float2 nax = f2(r0.x);
    // kx = x - ax for the lane's 8 columns: exact small integers (one FADD2 per column pair)
    // column pair jp lies in column half jp >> 1 (halves: slots 0-3 left, 4-7 right)
    auto live = [&](int jp) { return !use_halves<FWD_STRIP>() || ((HSEL >> (jp >> 1)) & 1); };
    float2 kx[FWD_STRIP / 2];
#pragma unroll
    for (int jp = 0; jp < FWD_STRIP / 2; ++jp)
        if (live(jp)) kx[jp] = __fadd2_rn(xj[jp], nax);
    bool cin[FWD_STRIP];
    unsigned rin = 0u;
    if (!FULL) {
        const unsigned cm = mw.x >> xo;
#pragma unroll
        for (int j = 0; j < FWD_STRIP; ++j) cin[j] = (cm >> colx<FWD_STRIP>(j)) & 1u;
        rin = mw.y >> yo;
    }
    const float2 cr = f2(r1.w), cg = f2(r2.x), cb = f2(r2.y);
    float dy = fmaf(yf0 - r0.y, invs, -r0.z);
#pragma unroll
    for (int r = 0; r < FWD_ROWS; ++r) {
        if (r > 0) dy += invs;                               // consecutive rows: exact to 1 ulp(1/s)
        const float v = r1.z * dy;                           // c1 dy
        float u = -(v * v);
        if (!FULL) u = ((rin >> r) & 1u) ? u : -INFINITY;    // lane's row outside [y0, y1]
        const float tau = fmaf(r1.y, dy, r1.x);              // b1 dy - a1 dl_x
        const float2 T2 = f2(tau), U2 = f2(u);
#pragma unroll
        for (int jp = 0; jp < FWD_STRIP / 2; ++jp) {
            if (!live(jp)) continue;                         // compile-time skip
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
                                              float g3, float m2d, float xlf, float2 yrow,
                                              const int (&yi)[2],
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
        const float2 G1 = f2(r2.z), G2 = f2(r2.w), G3 = f2(g3), M2D = f2(m2d);   // m2d = -2D
        float2 w0 = make_float2(0.f, 0.f);
#pragma unroll
        for (int h = 0; h < STRIP / 4; ++h) {
            if (use_halves<STRIP>() && !((hmask >> h) & 1)) continue;   // compile-time skip
            // anchor column 16 h: w = D kx + T; the second anchor of a Gaussian that evaluates
            // both halves as w0 + 16 D (one FFMA2 instead of an FADD for kx and an FFMA2)
            float2 w;
            if (h == 0)
                w = __ffma2_rn(D2, f2(kx0), T);
            else if (use_halves<STRIP>() && (hmask & 1))
                w = __ffma2_rn(D2, f2((float)colx<STRIP>(4 * h)), w0);
            else
                w = __ffma2_rn(D2, f2(kx0 + (float)colx<STRIP>(4 * h)), T);
            if (h == 0) w0 = w;
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

// Evaluation paths decided by the filter (one byte per staged record). Large configuration:
// MODE (0 masked, 1 direct, 2 recurrence) x column halves (both, left only, right only);
// small configuration: 0..2 full (no masks) x (both, left, right half), 3..5 masked likewise.
enum : int { P_REC3 = 0, P_REC1, P_REC2, P_DIR3, P_DIR1, P_DIR2, P_MSK3, P_MSK1, P_MSK2 };
constexpr int FRONT_PATH = 0;   // P_REC3 (large) / full over both halves (small configuration)

// records per warp buffer (> 32; a buffer is evaluated once it holds more than FWD_BUF - 32):
// 96 for the large tiles (48 -> 96: C5 forward -0.5%), 48 for the small ones (96: C2 +6%)
#ifndef GSR_FWD_BUF_LARGE
#define GSR_FWD_BUF_LARGE 96
#endif
#ifndef GSR_FWD_BUF_SMALL
#define GSR_FWD_BUF_SMALL 48
#endif
template <class CFG>
constexpr int fwd_buf() { return CFG::ROWS == 2 ? GSR_FWD_BUF_LARGE : GSR_FWD_BUF_SMALL; }
#ifndef GSR_FWD_SPLIT
#define GSR_FWD_SPLIT 1
#endif
#ifndef GSR_FWD_FRONT_UNROLL
#define GSR_FWD_FRONT_UNROLL 1
#endif
constexpr int kFrontUnroll = GSR_FWD_FRONT_UNROLL;
#ifndef GSR_FWD_CUTMASK
#define GSR_FWD_CUTMASK 1         // mask only the window edges that cut the support box
#endif
#ifndef GSR_FWD_HALVES
#define GSR_FWD_HALVES 1          // skip the column half a Gaussian's support misses
#endif

template <class CFG>
struct FwdSmem2 {
    static constexpr int FWD_BUF = fwd_buf<CFG>();
    struct PerWarp {
        float2 tot[FwdAcc<CFG>::NACC][32];                 // the warp's image (epilogue)
    };
    union {                       // the epilogue's buffers reuse the main loop's record buffers
        float4 rec[CFG::WARPS][2][FWD_BUF * REC_F4];      // staged records (main loop)
        struct {
            PerWarp wp[CFG::WARPS];                        // written after every warp's loop
            float stage[CFG::TH][CFG::TW * 3];             // HWC tile
        };
    };
    uint8_t path[CFG::WARPS][2][FWD_BUF];
    // window masks of the staged masked-path records (small configuration only, fwd_gauss)
    uint2 mw[CFG::WARPS][2][CFG::ROWS == 1 ? FWD_BUF : 1];
    CandChunk chunk;                                        // candidate stream table
};

// Stores the tile from the HWC staging area (every thread), with the fused L1 loss.
template <bool LOSS, class CFG>
__device__ __forceinline__ void fwd_store(const float (*stage)[CFG::TW * 3], const DevImg& im,
                                          int Tx0, int Ty0, float* __restrict__ out,
                                          const float* __restrict__ gt,
                                          double* __restrict__ loss_acc) {
    constexpr int TW = CFG::TW, TH = CFG::TH, ROWF = TW * 3;
    const int nx = min(TW, im.Ws - Tx0), ny = min(TH, im.row_end - Ty0);
    float l1 = 0.f;
    if (im.io != 0) {                                   // NEXT-4 formats (bf16 / planar CHW)
        for (int i = threadIdx.x; i < ny * nx * 3; i += (CFG::WARPS * 32)) {
            const int r = i / (nx * 3), c = i % (nx * 3);
            img_store(out, im, img_index(im, Ty0 + r, Tx0 + c / 3, c % 3), stage[r][c]);
        }
        return;
    }
    for (int r = threadIdx.x / 32; r < ny; r += CFG::WARPS) {   // one warp per row, coalesced
        const int lane = threadIdx.x & 31;
        const long long o = im.out_off + ((long long)(r + Ty0 - im.row_begin) * im.Ws + Tx0) * 3;
        const int nf = nx * 3;
        // whole rows as float4 where the row starts on a 16-B boundary of the caller's buffer
        // (the ABI does not require `out` / `gt` themselves to be 16-B aligned)
        const uintptr_t al = reinterpret_cast<uintptr_t>(out + o) |
                             (LOSS ? reinterpret_cast<uintptr_t>(gt + o) : uintptr_t(0));
        if (nx == TW && (al & 15) == 0) {
            for (int c4 = lane; c4 < ROWF / 4; c4 += 32) {
                const float4 v = *reinterpret_cast<const float4*>(&stage[r][4 * c4]);
                *reinterpret_cast<float4*>(out + o + 4 * c4) = v;
                if (LOSS) {
                    const float4 t = *reinterpret_cast<const float4*>(gt + o + 4 * c4);
                    l1 += fabsf(v.x - t.x) + fabsf(v.y - t.y) + fabsf(v.z - t.z) +
                          fabsf(v.w - t.w);
                }
            }
        } else {
            for (int c = lane; c < nf; c += 32) {
                const float v = stage[r][c];
                out[o + c] = v;
                if (LOSS) l1 += fabsf(v - gt[o + c]);
            }
        }
    }
    if (LOSS) {
        double d = (double)l1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        if ((threadIdx.x & 31) == 0 && d != 0.0) atomicAdd(loss_acc, d);
    }
}

// Sum the per-warp images (warp order, deterministic) into the HWC staging tile; reduce the
// split-K cluster CTAs' tiles through DSMEM in rank order; store (rank 0).
template <int KS, bool LOSS, class CFG>
__device__ __forceinline__ void fwd_epilogue(FwdSmem2<CFG>& sm, const DevImg& im, int Tx0,
                                             int Ty0, int krank, float* __restrict__ out,
                                             const float* __restrict__ gt,
                                             double* __restrict__ loss_acc) {
    constexpr int STRIP = CFG::STRIP, ROWS = CFG::ROWS, NACC = FwdAcc<CFG>::NACC;
    __syncthreads();                                   // every warp's image + no record reads
    for (int i = threadIdx.x; i < NACC * 32; i += (CFG::WARPS * 32)) {
        const int a = i >> 5, l = i & 31;
        float2 v = sm.wp[0].tot[a][l];
#pragma unroll
        for (int q = 1; q < CFG::WARPS; ++q) v = __fadd2_rn(v, sm.wp[q].tot[a][l]);
        const int xl = lane_x0<STRIP>(l), yl = ROWS * (l >> 2);
        const int k = a % 3;
        if constexpr (ROWS == 2) {                     // pair = (row 0, row 1) of column slot j
            const int x = xl + colx<STRIP>(a / 3);
            sm.stage[yl][3 * x + k] = v.x;
            sm.stage[yl + 1][3 * x + k] = v.y;
        } else {                                       // pair = two adjacent columns of one row
            const int jp = (a / 3) % (STRIP / 2), r = (a / 3) / (STRIP / 2);
            const int x = xl + colx<STRIP>(2 * jp);         // + 1: the pair's second column
            sm.stage[yl + r][3 * x + k] = v.x;
            sm.stage[yl + r][3 * (x + 1) + k] = v.y;
        }
    }
    if (KS > 1) {
        cluster_sync_all();                            // every CTA's tile is staged
        if (krank == 0) {
            float* st = &sm.stage[0][0];
            for (int i = threadIdx.x; i < CFG::TH * CFG::TW * 3; i += (CFG::WARPS * 32)) {
                float v = st[i];
                for (int q = 1; q < KS; ++q) v += ld_dsmem_f(st + i, q);
                st[i] = v;
            }
        }
        cluster_sync_all();                            // peers' staging read; rank 0's written
        if (krank != 0) return;
    } else {
        __syncthreads();
    }
    fwd_store<LOSS, CFG>(sm.stage, im, Tx0, Ty0, out, gt, loss_acc);
}

// The filter's decision for one candidate of a forward tile (columns fx0..fx1, rows fy0..fyc
// inside the image / band): keep = its support rect (R21) meets the tile; pth = its evaluation
// path; mwd = the window rect as tile column / row bit masks (small tiles' masked path). Shared
// by K4 and the debug lists.
template <class CFG>
__device__ __forceinline__ void fwd_classify(const int4 rc, int cl, int fx0, int fx1, int fy0,
                                             int fyc, bool& keep, int& pth, uint2& mwd) {
    constexpr int FTILE_H = CFG::TH, FWD_ROWS = CFG::ROWS, FWD_STRIP = CFG::STRIP;
    const unsigned sxs = (unsigned)rc.x, sys = (unsigned)rc.y;
    const int sx0 = (int)(sxs & 0xffffu), sx1 = (int)(sxs >> 16);
    const int sy0 = (int)(sys & 0xffffu), sy1 = (int)(sys >> 16);
    const int fy1 = fy0 + FTILE_H - 1;                 // the tile's last row (unclipped)
    keep = !(sx1 < fx0 || sx0 > fx1 || sy1 < fy0 || sy0 > fyc);
    const unsigned xs = (unsigned)rc.z, ys = (unsigned)rc.w;
    const int x0 = (int)(xs & 0xffffu), x1 = (int)(xs >> 16);
    const int y0 = (int)(ys & 0xffffu), y1 = (int)(ys >> 16);
    bool full;
    if (FWD_ROWS == 1 && GSR_FWD_CUTMASK) {
        // small tiles (narrow windows, where the window often cuts the support): the mask
        // matters only on a side where the window edge lies inside the tile AND cuts the
        // +-13.5 sigma box (the support ends at the window edge); where the support edge lies
        // inside the window, every pixel beyond it is outside the box and evaluates to exactly
        // 0 (R21). C2 -3%; the large tiles keep the plain test (their windows rarely end inside
        // a tile)
        full = !((x0 > fx0 && sx0 == x0) || (x1 < fx1 && sx1 == x1) ||
                 (y0 > fy0 && sy0 == y0) || (y1 < fy1 && sy1 == y1));
    } else {
        full = x0 <= fx0 && x1 >= fx1 && y0 <= fy0 && y1 >= fy1;
    }
    // column halves the support meets (left 16 / right 16 columns)
    const bool hl = sx0 <= fx0 + 15, hr = sx1 >= fx0 + 16;
    const int hv = !GSR_FWD_HALVES || !use_halves<FWD_STRIP>() || (hl && hr) ? 0 : (hl ? 1 : 2);
    if constexpr (FWD_ROWS == 2) {
        pth = (full ? ((cl & 1) ? P_REC3 : P_DIR3) : P_MSK3) + hv;
    } else {
        pth = (full ? 0 : 3) + hv;
        const int c0 = max(x0 - fx0, 0), c1 = min(x1 - fx0, 31);
        const int w0 = max(y0 - fy0, 0), w1 = min(y1 - fy0, 31);
        mwd.x = c1 < c0 ? 0u : (unsigned)(((2ull << c1) - 1ull) & ~((1ull << c0) - 1ull));
        mwd.y = w1 < w0 ? 0u : (unsigned)(((2ull << w1) - 1ull) & ~((1ull << w0) - 1ull));
    }
}

template <int KS, bool LOSS, class CFG>
__global__ void __launch_bounds__(CFG::WARPS * 32, 16 / CFG::WARPS) k_render_fwd2(const ImgTable tab,
                                                              const float4* __restrict__ rec,
                                                              const int4* __restrict__ rects,
                                                              const uint8_t* __restrict__ cls,
                                                              const int* __restrict__ cell_start,
                                                              const int* __restrict__ ext,
                                                              const int2* __restrict__ reach,
                                                              float* __restrict__ out,
                                                              const float* __restrict__ gt,
                                                              double* __restrict__ loss_acc) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    FwdSmem2<CFG>& sm = *reinterpret_cast<FwdSmem2<CFG>*>(smem_raw);
    constexpr int FWD_BUF = fwd_buf<CFG>();
    constexpr int FTILE_W = CFG::TW, FTILE_H = CFG::TH, FWD_STRIP = CFG::STRIP,
                  FWD_ROWS = CFG::ROWS, NACC = FwdAcc<CFG>::NACC;

    const int tile = blockIdx.x / KS;
    const int krank = KS > 1 ? (int)cluster_rank() : 0;
    const int kimg = find_image_by_sftile(tab, tile);
    const DevImg& im = tab.img[kimg];
    const int t = tile - im.sftile_base;
    const int Tx0 = (t % im.fntx) * FTILE_W;
    const int Ty0 = im.row_begin + (t / im.fntx) * FTILE_H;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    const int fx0 = Tx0, fx1 = min(Tx0 + FTILE_W - 1, im.Ws - 1);   // tile footprint
    const int fy0 = Ty0, fy1 = min(Ty0 + FTILE_H - 1, im.row_end - 1);
    const float invs = im.invsy;     // rows: dy = (y - ay)/sy - dl_y

    // lane geometry (every warp covers the whole tile)
    const int xo = lane_x0<FWD_STRIP>(lane), yo = FWD_ROWS * (lane >> 2);   // in the tile
    const int xl0 = Tx0 + xo;
    const int yl0 = Ty0 + yo;
    float2 xj[FWD_STRIP / 2];
#pragma unroll
    for (int jp = 0; jp < FWD_STRIP / 2; ++jp)
        xj[jp] = make_float2((float)(xl0 + colx<FWD_STRIP>(2 * jp)),
                             (float)(xl0 + colx<FWD_STRIP>(2 * jp + 1)));
    const float xlf = (float)xl0;
    const float2 yrow = make_float2((float)yl0, (float)(yl0 + 1));
    int yi[FWD_ROWS];
#pragma unroll
    for (int r = 0; r < FWD_ROWS; ++r) yi[r] = yl0 + r;
    const float yf0 = (float)yl0;

    const bool live = fy0 <= fy1;
    CandStream vs;
    vs.cs = cell_start;
    vs.reach = reach;
    vs.row0 = im.cell_base;
    vs.row_stride = im.ncx;
    vs.cx_lo = (Tx0 - query_ext(ext, kimg, 0) + 1 + im.offx) / CELL;
    vs.cx_hi = min(im.ncx - 1, (fx1 + im.offx) / CELL);
    vs.cy_hi = min(im.ncy - 1, (fy1 - im.row_begin + im.offy) / CELL);
    vs.X0 = fx0;
    vs.Y0 = fy0;
    vs.trim = im.dense && vs.cx_hi - vs.cx_lo + 1 >= 6;
    const int cy_first = (Ty0 - im.row_begin - query_ext(ext, kimg, 1) + 1 + im.offy) / CELL;
    if (warp == 0) vs.build(sm.chunk, live ? cy_first : vs.cy_hi + 1, lane);
    __syncthreads();
    int ctotal = sm.chunk.pre[32], r0 = 0, round = 0;
    const unsigned lt = (1u << lane) - 1u;
    // candidate batches in flight: batch 0 is filtered while batches 1 .. SD-1 load
    constexpr int SD = GSR_FWD_SCAN_D;
    int nb[SD], sb[SD];                 // candidates in the batch, the lane's candidate position
    int4 rb[SD];
    int cb[SD];
    // positions: the P = KS W parts (the warps of the split-K cluster) interleave at the lane
    // level, part p = krank W + w takes positions p, p + P, p + 2P, ... (CandStream): the kept
    // candidates cluster along the stream (the cells nearest the tile), and the interleave
    // gives every warp and every cluster CTA an even share of each cluster, with a fixed,
    // deterministic assignment (whole batches per warp left one warp waiting at the epilogue
    // for up to 20% of the samples at C4)
    constexpr int NPARTS = KS * CFG::WARPS;
    const int part = krank * CFG::WARPS + warp;
    auto fetch = [&](int j) {
        nb[j] = 0;
        sb[j] = 0;
        while (ctotal > 0) {
            const int base = 32 * NPARTS * round;
            if (base + part < ctotal) {
                ++round;
                nb[j] = min(32, (ctotal - base - part + NPARTS - 1) / NPARTS);
                while (base >= sm.chunk.pre[r0 + 1]) ++r0;
                const int v = base + NPARTS * lane + part;
                if (v < ctotal) sb[j] = cand_index(sm.chunk, v, r0);
                break;
            }
            // chunk exhausted by this warp: once every warp is here, warp 0 builds the next one
            // (every warp walks the same chunk sequence, so the barriers match)
            if (sm.chunk.cy_next > vs.cy_hi) break;
            __syncthreads();
            if (warp == 0) vs.build(sm.chunk, sm.chunk.cy_next, lane);
            __syncthreads();
            ctotal = sm.chunk.pre[32];
            r0 = 0;
            round = 0;
        }
        rb[j] = make_int4(0xffff, 0, 0, 0);     // no candidate: a support rect no tile meets
        cb[j] = 0;
        if (lane < nb[j]) {
            rb[j] = __ldg(rects + sb[j]);
            cb[j] = __ldg(cls + sb[j]);
        }
    };

    // one register accumulator per lane for the whole tile
    float2 acc[NACC];
#pragma unroll
    for (int a = 0; a < NACC; ++a) acc[a] = make_float2(0.f, 0.f);

    // A staged buffer holds the Gaussians of the front path (the most common one: the
    // recurrence over both column halves, or the unmasked small-tile path) at slots 0, 1, ...
    // and every other path from slot FWD_BUF - 1 downwards (GSR_FWD_SPLIT): the front run is
    // evaluated without any per-Gaussian dispatch.
    auto process_front = [&](int pbuf, int nf) {
        const float4* q = &sm.rec[warp][pbuf][0];
#ifdef GSR_DIAG_FWD_NOEVAL
        if (nf > 0) nf = q[0].x == 12345.f ? 1 : 0;
#endif
        // one 32-bit shared address as the loop variable and the load base (a generic pointer
        // kept a second register and an add per Gaussian)
        uint32_t a = smem_u32(q);
        const uint32_t ae = a + (uint32_t)(16 * REC_F4 * nf);
#pragma unroll kFrontUnroll
        for (; a != ae; a += 16 * REC_F4) {
            const float4 r0 = lds_f4(a), r1 = lds_f4(a + 16), r2 = lds_f4(a + 32);
            if constexpr (FWD_ROWS == 2) {
                const float4 r3 = lds_f4(a + 48);
                const float4 r2g = make_float4(r2.x, r2.y, r3.x, r3.y);
                fwd_gauss_r2h<2, FWD_STRIP, 3>(r0, r1, r2g, r3.z, r3.w, xlf, yrow, yi, xl0, invs, acc);
            } else {
                fwd_gauss<CFG, true, 3>(r0, r1, r2, make_uint2(0u, 0u), xj, yf0, xo, yo, invs, acc);
            }
        }
    };
    auto process = [&](int pbuf, int pbeg, int pcnt) {
        const float4* sr = &sm.rec[warp][pbuf][0];
        const uint8_t* pp = &sm.path[warp][pbuf][0];
        const uint2* mws = &sm.mw[warp][pbuf][0];
#ifdef GSR_DIAG_FWD_NOEVAL       // timing diagnostic only (wrong results): no evaluation
        if (pcnt > pbeg) pcnt = sr[0].x == 12345.f ? pbeg + 1 : pbeg;
#endif
        if constexpr (FWD_ROWS == 1 && !use_halves<FWD_STRIP>()) {
            if (GSR_FWD_SPLIT) {          // the small tiles' other path is the masked one
                uint32_t qa = smem_u32(sr) + (uint32_t)(16 * REC_F4 * pbeg);
                for (int g = pbeg; g < pcnt; ++g, qa += 16 * REC_F4)
                    fwd_gauss<CFG, false, 3>(lds_f4(qa), lds_f4(qa + 16), lds_f4(qa + 32), mws[g],
                                             xj, yf0, xo, yo, invs, acc);
                return;
            }
        }
        int pnext = pcnt > pbeg ? pp[pbeg] : 0;
        uint32_t ra = smem_u32(sr) + (uint32_t)(16 * REC_F4 * pbeg);   // record g's address
        for (int g = pbeg; g < pcnt; ++g, ra += 16 * REC_F4) {
#ifdef GSR_DIAG_FWD_NOMASK       // timing diagnostic only (wrong results): masked -> full paths
            const int pth = FWD_ROWS == 2 ? (pnext >= P_MSK3 ? pnext - 3 : pnext) : (pnext >= 3 ? pnext - 3 : pnext);
#else
            const int pth = pnext;
#endif
            if (g + 1 < pcnt) pnext = pp[g + 1];          // next Gaussian's path, one ahead
            const float4 r0 = lds_f4(ra), r1 = lds_f4(ra + 16), r2 = lds_f4(ra + 32);
            if constexpr (FWD_ROWS == 2) {
                // the back's common paths first: the single-half recurrences (P_REC3 is only
                // here without GSR_FWD_SPLIT)
                if ((unsigned)(pth - P_REC1) <= (unsigned)(P_REC2 - P_REC1) || pth == P_REC3) {
                    const float4 r3 = lds_f4(ra + 48);
                    const float4 r2g = make_float4(r2.x, r2.y, r3.x, r3.y);
                    if (pth == P_REC1)
                        fwd_gauss_r2h<2, FWD_STRIP, 1>(r0, r1, r2g, r3.z, r3.w, xlf, yrow, yi, xl0, invs, acc);
                    else if (pth == P_REC2)
                        fwd_gauss_r2h<2, FWD_STRIP, 2>(r0, r1, r2g, r3.z, r3.w, xlf, yrow, yi, xl0, invs, acc);
                    else
                        fwd_gauss_r2h<2, FWD_STRIP, 3>(r0, r1, r2g, r3.z, r3.w, xlf, yrow, yi, xl0, invs, acc);
                } else if (pth >= P_MSK3) {
                    if (pth == P_MSK3)
                        fwd_gauss_r2h<0, FWD_STRIP, 3>(r0, r1, r2, 0.f, 0.f, xlf, yrow, yi, xl0, invs, acc);
                    else if (pth == P_MSK1)
                        fwd_gauss_r2h<0, FWD_STRIP, 1>(r0, r1, r2, 0.f, 0.f, xlf, yrow, yi, xl0, invs, acc);
                    else
                        fwd_gauss_r2h<0, FWD_STRIP, 2>(r0, r1, r2, 0.f, 0.f, xlf, yrow, yi, xl0, invs, acc);
                } else {
                    if (pth == P_DIR3)
                        fwd_gauss_r2h<1, FWD_STRIP, 3>(r0, r1, r2, 0.f, 0.f, xlf, yrow, yi, xl0, invs, acc);
                    else if (pth == P_DIR1)
                        fwd_gauss_r2h<1, FWD_STRIP, 1>(r0, r1, r2, 0.f, 0.f, xlf, yrow, yi, xl0, invs, acc);
                    else
                        fwd_gauss_r2h<1, FWD_STRIP, 2>(r0, r1, r2, 0.f, 0.f, xlf, yrow, yi, xl0, invs, acc);
                }
            } else {   // 0..2 full (both / left / right half), 3..5 masked
                if (pth == 0) fwd_gauss<CFG, true, 3>(r0, r1, r2, make_uint2(0u, 0u), xj, yf0, xo, yo, invs, acc);
                else if (pth == 1) fwd_gauss<CFG, true, 1>(r0, r1, r2, make_uint2(0u, 0u), xj, yf0, xo, yo, invs, acc);
                else if (pth == 2) fwd_gauss<CFG, true, 2>(r0, r1, r2, make_uint2(0u, 0u), xj, yf0, xo, yo, invs, acc);
                else if (pth == 3) fwd_gauss<CFG, false, 3>(r0, r1, r2, mws[g], xj, yf0, xo, yo, invs, acc);
                else if (pth == 4) fwd_gauss<CFG, false, 1>(r0, r1, r2, mws[g], xj, yf0, xo, yo, invs, acc);
                else fwd_gauss<CFG, false, 2>(r0, r1, r2, mws[g], xj, yf0, xo, yo, invs, acc);
            }
        }
    };

#pragma unroll
    for (int d = 0; d < SD; ++d) fetch(d);
    // cnt / pend: front-path entries of the filling / pending buffer, cntb / pendb: the rest
    int b = 0, cnt = 0, pend = -1, cntb = 0, pendb = 0;
    auto run = [&](int buf, int nf, int nbk) {
        if (GSR_FWD_SPLIT) {
            process_front(buf, nf);
            process(buf, FWD_BUF - nbk, FWD_BUF);
        } else {
            process(buf, 0, nf);
        }
    };
    while (true) {
        const bool end = nb[0] == 0;
        if (!end) {
            bool keep = false;
            int pth = 0;
            uint2 mwd = make_uint2(0u, 0u);
            // every lane (lanes past the batch hold the empty sentinel rect)
            fwd_classify<CFG>(rb[0], cb[0], fx0, fx1, fy0, fy1, keep, pth, mwd);
#if GSR_FWD_SPLIT
            const bool front = keep && pth == FRONT_PATH;
            const unsigned mf = __ballot_sync(0xffffffffu, front);
            const unsigned mb = __ballot_sync(0xffffffffu, keep && !front);
            if (keep) {
                const int slot = front ? cnt + __popc(mf & lt)
                                       : FWD_BUF - 1 - (cntb + __popc(mb & lt));
                GSR_CHECK(slot >= 0 && slot < FWD_BUF && cnt + cntb + __popc(mf | mb) <= FWD_BUF);
                GSR_CHECK(sb[0] >= 0 && sb[0] < cell_start[tab.total_cells]);
                sm.path[warp][b][slot] = (uint8_t)pth;
                if constexpr (FWD_ROWS == 1) sm.mw[warp][b][slot] = mwd;
                const float4* src = rec + (long long)REC_F4 * sb[0];
                float4* dst = &sm.rec[warp][b][REC_F4 * slot];
#pragma unroll
                for (int q = 0; q < REC_F4; ++q) cp_async16(dst + q, src + q);
            }
            cnt += __popc(mf);
            cntb += __popc(mb);
#else
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const int slot = cnt + __popc(m & lt);
                sm.path[warp][b][slot] = (uint8_t)pth;
                if constexpr (FWD_ROWS == 1) sm.mw[warp][b][slot] = mwd;
                const float4* src = rec + (long long)REC_F4 * sb[0];
                float4* dst = &sm.rec[warp][b][REC_F4 * slot];
#pragma unroll
                for (int q = 0; q < REC_F4; ++q) cp_async16(dst + q, src + q);
            }
            cnt += __popc(m);
#endif
#pragma unroll
            for (int d = 0; d + 1 < SD; ++d) {
                nb[d] = nb[d + 1]; sb[d] = sb[d + 1]; rb[d] = rb[d + 1]; cb[d] = cb[d + 1];
            }
            fetch(SD - 1);
        }
        // a full buffer (or the last one) is committed; the OTHER buffer, whose copies are
        // older, is evaluated meanwhile -- at the end, the last one after all copies landed
        // (one evaluation call site: the evaluation code is inlined once)
        const bool fl = cnt + cntb > FWD_BUF - 32 || (end && cnt + cntb > 0);
        if (fl) cp_async_commit();
        if (fl || end) {
            if (pend >= 0) {
                if (fl) cp_async_wait<1>(); else cp_async_wait<0>();
                __syncwarp();
                run(b ^ 1, pend, pendb);
                __syncwarp();
            }
            pend = -1;
            if (fl) {
                pend = cnt;
                pendb = cntb;
                b ^= 1;
                cnt = 0;
                cntb = 0;
            }
        }
        if (end && pend < 0) break;
    }
    __syncthreads();                                   // every warp is done with the records
#pragma unroll
    for (int a = 0; a < NACC; ++a) sm.wp[warp].tot[a][lane] = acc[a];   // (after the barrier)
    fwd_epilogue<KS, LOSS, CFG>(sm, im, Tx0, Ty0, krank, out, gt, loss_acc);
}

// Materialised forward tile lists (test-only, gsr_debug_fwd_tile_lists): one warp per forward
// tile in image order walks the tile's candidate stream exactly as K4 does (CandStream::build,
// cand_index) and applies K4's filter decision (fwd_classify); the kept candidates' Gaussian
// indices and paths in stream order. offs == nullptr: counts only.
template <class CFG>
__global__ void __launch_bounds__(32) k_debug_fwd_lists(
    const ImgTable tab, const int4* __restrict__ rects, const uint8_t* __restrict__ cls,
    const int* __restrict__ cell_start, const int* __restrict__ ext,
    const int2* __restrict__ reach, const int* __restrict__ perm, const int* __restrict__ offs,
    int* __restrict__ counts, int* __restrict__ ids, uint8_t* __restrict__ paths) {
    __shared__ CandChunk ch;
    const int tile = blockIdx.x, lane = threadIdx.x;
    const int kimg = find_image_by_ftile(tab, tile);
    const DevImg& im = tab.img[kimg];
    const int t = tile - im.ftile_base;
    const int Tx0 = (t % im.fntx) * CFG::TW;
    const int Ty0 = im.row_begin + (t / im.fntx) * CFG::TH;
    const int fx0 = Tx0, fx1 = min(Tx0 + CFG::TW - 1, im.Ws - 1);
    const int fy0 = Ty0, fy1 = min(Ty0 + CFG::TH - 1, im.row_end - 1);
    CandStream vs;
    vs.cs = cell_start;
    vs.reach = reach;
    vs.row0 = im.cell_base;
    vs.row_stride = im.ncx;
    vs.cx_lo = (Tx0 - query_ext(ext, kimg, 0) + 1 + im.offx) / CELL;
    vs.cx_hi = min(im.ncx - 1, (fx1 + im.offx) / CELL);
    vs.cy_hi = min(im.ncy - 1, (fy1 - im.row_begin + im.offy) / CELL);
    vs.X0 = fx0;
    vs.Y0 = fy0;
    vs.trim = im.dense && vs.cx_hi - vs.cx_lo + 1 >= 6;
    int cy = fy0 <= fy1 ? (Ty0 - im.row_begin - query_ext(ext, kimg, 1) + 1 + im.offy) / CELL
                        : vs.cy_hi + 1;
    const int base = offs ? offs[tile] : 0;
    int c = 0;
    while (true) {
        vs.build(ch, cy, lane);
        __syncwarp();
        const int total = ch.pre[32];
        for (int v0 = 0; v0 < total; v0 += 32) {
            const int v = v0 + lane;
            bool keep = false;
            int pth = 0, p = 0;
            uint2 mwd = make_uint2(0u, 0u);
            if (v < total) {
                p = cand_index(ch, v, 0);
                fwd_classify<CFG>(rects[p], cls[p], fx0, fx1, fy0, fy1, keep, pth, mwd);
            }
            const unsigned m = __ballot_sync(0xffffffffu, keep);
            if (keep && offs) {
                const int o = base + c + __popc(m & ((1u << lane) - 1u));
                ids[o] = perm[p];
                paths[o] = (uint8_t)pth;
            }
            c += __popc(m);
        }
        __syncwarp();
        if (ch.cy_next > vs.cy_hi) break;
        cy = ch.cy_next;
    }
    if (!offs && lane == 0) counts[tile] = c;
}

// Per-device one-time setup of an instance (the dynamic shared-memory opt-in is a property of
// the function on the CURRENT device; also loads its code under CUDA lazy loading).
constexpr int MAX_DEVICES = 64;
inline int current_device() {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= MAX_DEVICES) d = 0;
    return d;
}
template <int KS, bool LOSS, class CFG>
cudaError_t fwd2_prepare() {
    static std::atomic<bool> attr_set[MAX_DEVICES];   // concurrent first calls repeat the set
    const int d = current_device();
    if (!attr_set[d].load(std::memory_order_acquire)) {
        cudaError_t e = cudaFuncSetAttribute(k_render_fwd2<KS, LOSS, CFG>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)sizeof(FwdSmem2<CFG>));
        if (e != cudaSuccess) return e;
        attr_set[d].store(true, std::memory_order_release);
    }
    return cudaSuccess;
}

template <int KS, bool LOSS, class CFG>
cudaError_t launch_ks3(const ImgTable& tab, const Workspace& ws, float* out, const float* gt,
                       double* loss_acc, cudaStream_t st) {
    const size_t smem = sizeof(FwdSmem2<CFG>);
    cudaError_t e0 = fwd2_prepare<KS, LOSS, CFG>();
    if (e0 != cudaSuccess) return e0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)tab.total_ftiles * KS);
    cfg.blockDim = dim3((CFG::WARPS * 32));
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
                              (const int4*)ws.rects, (const uint8_t*)ws.cls,
                              (const int*)ws.cell_start, (const int*)ws.ext,
                              (const int2*)ws.reach, out, gt, loss_acc);
}

template <int KS, bool LOSS>
cudaError_t launch_ks2(const ImgTable& tab, const Workspace& ws, float* out, const float* gt,
                       double* loss_acc, cudaStream_t st) {
    return tab.fwd_small ? launch_ks3<KS, LOSS, FwdCfgSmall>(tab, ws, out, gt, loss_acc, st)
                         : launch_ks3<KS, LOSS, FwdCfgWide>(tab, ws, out, gt, loss_acc, st);
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
    const auto k = k_render_fwd2<1, false, CFG>;
    const size_t smem = sizeof(FwdSmem2<CFG>);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    return resident_slots(k, (CFG::WARPS * 32), smem);
}

}  // namespace

cudaError_t launch_render_fwd(const ImgTable& tab, const Workspace& ws, float* out,
                              cudaStream_t st, const float* gt, double* loss_acc) {
    if (tab.total_ftiles <= 0) return cudaSuccess;
    count_launches(1);
    int h = prof_begin(1, st);
    // every instance the split choice can pick is set up (and its code loaded) on the first
    // call on a device, so a later batch with a new split factor does not pay a module load
    static std::once_flag prepared[MAX_DEVICES];
    const int dev = current_device();
    std::call_once(prepared[dev], [] {
        fwd2_prepare<1, false, FwdCfgSmall>(); fwd2_prepare<2, false, FwdCfgSmall>();
        fwd2_prepare<4, false, FwdCfgSmall>(); fwd2_prepare<8, false, FwdCfgSmall>();
        fwd2_prepare<1, true, FwdCfgSmall>(); fwd2_prepare<2, true, FwdCfgSmall>();
        fwd2_prepare<4, true, FwdCfgSmall>(); fwd2_prepare<8, true, FwdCfgSmall>();
        fwd2_prepare<1, false, FwdCfgWide>(); fwd2_prepare<2, false, FwdCfgWide>();
        fwd2_prepare<4, false, FwdCfgWide>(); fwd2_prepare<8, false, FwdCfgWide>();
        fwd2_prepare<1, true, FwdCfgWide>(); fwd2_prepare<2, true, FwdCfgWide>();
        fwd2_prepare<4, true, FwdCfgWide>(); fwd2_prepare<8, true, FwdCfgWide>();
    });
    static std::atomic<int> slots_small[MAX_DEVICES], slots_wide[MAX_DEVICES];
    std::atomic<int>& sl = tab.fwd_small ? slots_small[dev] : slots_wide[dev];
    int slots = sl.load(std::memory_order_relaxed);
    if (slots == 0) {
        slots = tab.fwd_small ? fwd_slots<FwdCfgSmall>() : fwd_slots<FwdCfgWide>();
        sl.store(slots, std::memory_order_relaxed);
    }
#ifdef GSR_FORCE_KS_FWD                 // A/B builds only
    const int ks = GSR_FORCE_KS_FWD;
#else
    const int ks = split_k_factor(tab.total_ftiles, slots);
#endif
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

cudaError_t launch_debug_fwd_lists(const ImgTable& tab, const Workspace& ws, const int* perm,
                                   const int* offs, int* counts, int* ids, uint8_t* paths,
                                   cudaStream_t st) {
    if (tab.total_ftiles <= 0) return cudaSuccess;
    if (tab.fwd_small)
        k_debug_fwd_lists<FwdCfgSmall><<<tab.total_ftiles, 32, 0, st>>>(
            tab, ws.rects, ws.cls, ws.cell_start, ws.ext, ws.reach, perm, offs, counts, ids, paths);
    else
        k_debug_fwd_lists<FwdCfgWide><<<tab.total_ftiles, 32, 0, st>>>(
            tab, ws.rects, ws.cls, ws.cell_start, ws.ext, ws.reach, perm, offs, counts, ids, paths);
    return cudaGetLastError();
}

}  // namespace gsr
