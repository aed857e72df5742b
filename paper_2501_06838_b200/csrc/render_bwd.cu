// render_bwd.cu -- K5 (backward pair pass -> per-Gaussian moments) and K6 (finalize).
//
// Notation (Eq. 2): u = dx/sx, v = dy/sy, D = 1 - rho^2, Q = (u^2 - 2 rho u v +
// v^2)/D = p^2/D + v^2 with p = u - rho v. The kernels work in the scaled coordinates of the
// factored exponent, wq = sqrt(k/D) p and vq = sqrt(k) v (k = log2(e)/2), so 2^(-(wq^2+vq^2))
// = exp(-Q/2). For L with upstream gradient g = dL/dI every pair (Gaussian i, pixel (x,y))
// inside the window contributes, with e = exp(-Q/2), c' = alpha c K, w = e (g . c'):
//   m0..2 += e g_k,  m3 += w wq,  m4 += w vq,  m5 += w wq^2,  m6 += w wq vq,  m7 += w vq^2.
// The (p, v) basis keeps the finalize well conditioned as |rho| -> 1 (the (dx, dy) basis loses
// 1/sqrt(D) digits there). K6 (fp64), with S0 = sum w = alpha K (c . m012), Sp = m3/kp,
// Sv = m4/sqrt(k), Spp = m5/kp^2, Spv = m6/(kp sqrt(k)), Svv = m7/k, kp = sqrt(k/D):
//   d alpha = K (c . m012),  d c_k = alpha K m_k
//   d mu_x = Sp/(sx D),  d mu_y = (Sv - rho Sp/D)/sy
//   d sx = ((Spp + rho Spv)/D - S0)/sx,  d sy = (Svv - rho Spv/D - S0)/sy
//   d rho = (rho S0 + Spv - rho Spp/D)/D
// (derivation in DESIGN.md "Backward"; the oracle uses direct per-pair derivatives instead).
//
// Layout of K5: one CTA (4 warps) per 64 x 8 HR tile with the tile's dL/dI staged in shared
// memory as column pairs. Lanes own Gaussians: each warp scans its share of the tile's
// candidate spans (support rect vs tile; SCAN_U chunks of loads in flight), queues the hits with
// a key = their clipped column range; the CTA sorts the first <= 512 hits of every warp's queue
// together by key (GSR_BWD_CTASORT) and the warps evaluate its groups of 32 round-robin: all 32
// lanes of a group walk the same pixels (warp-uniform loop bounds from the union of their support
// rects), reading dL/dI as shared-memory broadcasts. Per-pair work is paired over two pixels with
// FFMA2. Within a row the vq-dependent moments are factored out (sum_row w vq = vq sum_row w, ...),
// so a pair costs 12.5 FP32 lane-ops + 1 ex2 (kx shared by a row pair, w, q, 3 e g, 3 g.c',
// 4 moments); lanes process two rows at once for two independent accumulation chains. Row
// partials (fp32, <= 32 terms per register half) are folded into fp32 per-(Gaussian, tile)
// accumulators, which leave the CTA as 8 fp64 atomics -- the only global atomics of the backward.
#include <atomic>

#include "gsr_internal.cuh"

#ifndef GSR_BWD_UNROLL
#define GSR_BWD_UNROLL 8
#endif
#ifndef GSR_BWD_SCAN_U
#define GSR_BWD_SCAN_U 4          // candidate chunks whose rect loads are in flight together
#endif
#ifndef GSR_BWD_KQ
#define GSR_BWD_KQ 16             // grouping key: column buckets per axis (8 or 16)
#endif
#ifndef GSR_BWD_BATCH
#define GSR_BWD_BATCH 512         // hits per sorted batch (multiple of 32)
#endif
#ifndef GSR_BWD_CTASORT
#define GSR_BWD_CTASORT 1
#endif
#ifndef GSR_BWD_MACC_T
#define GSR_BWD_MACC_T float      // per-(Gaussian, tile) accumulator type of the row folds
#endif

namespace gsr {

namespace {

constexpr int kBwdUnroll = GSR_BWD_UNROLL;
#ifndef GSR_BWD_UNROLL_MASKED
#define GSR_BWD_UNROLL_MASKED 4   // the masked column segments (window edges inside the union;
                                  // C2 -2%, C4/C5 unchanged; 2: +2% at C4/C5)
#endif
constexpr int kBwdUnrollMasked = GSR_BWD_UNROLL_MASKED;
constexpr int BWD_BATCH = GSR_BWD_BATCH;

__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }

struct LaneG {        // per-lane Gaussian constants
    float2 D2, cr, cg, cb;           // w = D kx + T_row (D = a1/s, T = b1 dy - a1 dl_x)
    int x0, x1;
};

struct RowAcc {       // per-row partial sums of a lane (register pairs = two pixels)
    float2 FR, FG, FB, W1, W2;
};

// Both rows of a row pair at one column pair, ordered so that every FFMA2 after the first of a
// group shares an operand register (same slot) with its predecessor: the operand then comes
// from the reuse cache and the instruction reads two fresh register pairs instead of three
// (register-file bank bandwidth: 2 instead of 3 issue cycles, tools/microbench.cu "ffma2_nr").
template <bool MASKED>
__device__ __forceinline__ void pix_pair2(const float4 gaA, const float4 gaB, const float4 gbb,
                                          const float2 kx, const float2 TA,
                                          const float2 UA, const float2 TB, const float2 UB,
                                          const LaneG& L, bool in0, bool in1, RowAcc& A,
                                          RowAcc& B) {
    const float2 wA = __ffma2_rn(L.D2, kx, TA);
    const float2 wB = __ffma2_rn(L.D2, kx, TB);
    float2 qA = __ffma2_rn(make_float2(-wA.x, -wA.y), wA, UA);
    float2 qB = __ffma2_rn(make_float2(-wB.x, -wB.y), wB, UB);
    if (MASKED) {
        qA.x = in0 ? qA.x : -INFINITY;
        qA.y = in1 ? qA.y : -INFINITY;
        qB.x = in0 ? qB.x : -INFINITY;
        qB.y = in1 ? qB.y : -INFINITY;
    }
    const float2 grA = make_float2(gaA.x, gaA.y), ggA = make_float2(gaA.z, gaA.w);
    const float2 grB = make_float2(gaB.x, gaB.y), ggB = make_float2(gaB.z, gaB.w);
    const float2 gbA = make_float2(gbb.x, gbb.y), gbB = make_float2(gbb.z, gbb.w);
    // g . c' of both rows, snake order (c' shared between rows, g between channels)
    float2 gcA = __fmul2_rn(grA, L.cr);
    float2 gcB = __fmul2_rn(grB, L.cr);
    gcB = __ffma2_rn(ggB, L.cg, gcB);
    gcA = __ffma2_rn(ggA, L.cg, gcA);
    gcA = __ffma2_rn(gbA, L.cb, gcA);
    gcB = __ffma2_rn(gbB, L.cb, gcB);
    const float2 eA = make_float2(ex2_approx(qA.x), ex2_approx(qA.y));
    const float2 eB = make_float2(ex2_approx(qB.x), ex2_approx(qB.y));
    // channel sums, snake: e shared within a row, g never shared -> e reuse
    A.FR = __ffma2_rn(eA, grA, A.FR);
    A.FG = __ffma2_rn(eA, ggA, A.FG);
    A.FB = __ffma2_rn(eA, gbA, A.FB);
    B.FB = __ffma2_rn(eB, gbB, B.FB);
    B.FG = __ffma2_rn(eB, ggB, B.FG);
    B.FR = __ffma2_rn(eB, grB, B.FR);
    // y = e (g . c'), W1 += y w' (an FADD2: two register pairs), W2 += (y w') w'
    const float2 ywA = __fmul2_rn(__fmul2_rn(eA, gcA), wA);
    const float2 ywB = __fmul2_rn(__fmul2_rn(eB, gcB), wB);
    A.W1 = __fadd2_rn(A.W1, ywA);
    A.W2 = __ffma2_rn(ywA, wA, A.W2);
    B.W1 = __fadd2_rn(B.W1, ywB);
    B.W2 = __ffma2_rn(ywB, wB, B.W2);
}

// Columns [c_begin, c_end) (pairs) of two rows at once: the column part (kx, masks, dL/dI
// addresses) is shared, and the two rows give two independent accumulation chains.
template <bool MASKED>
__device__ __forceinline__ void row2_pairs(int c_begin, int c_end, const float4* __restrict__ gA0,
                                           const float4* __restrict__ gA1,
                                           const float4* __restrict__ gBB, float kT,
                                           const LaneG& L, int Tx0, const float2 T0,
                                           const float2 U0, const float2 T1, const float2 U1,
                                           RowAcc& A0, RowAcc& A1) {
    float2 kx = make_float2(kT + (float)c_begin, kT + (float)(c_begin + 1));
    const float2 two = f2(2.0f);
    constexpr int UNR = MASKED ? kBwdUnrollMasked : kBwdUnroll;
#pragma unroll UNR
    for (int c = c_begin; c < c_end; c += 2) {
        const int cp = c >> 1;
        bool in0 = true, in1 = true;
        if (MASKED) {
            const int xa = Tx0 + c;
            in0 = xa >= L.x0 && xa <= L.x1;
            in1 = xa + 1 >= L.x0 && xa + 1 <= L.x1;
        }
        pix_pair2<MASKED>(gA0[cp], gA1[cp], gBB[cp], kx, T0, U0, T1, U1, L, in0, in1, A0, A1);
        kx = __fadd2_rn(kx, two);
    }
}

// fold one row's partials into the fp64 per-(Gaussian, tile) moments
typedef GSR_BWD_MACC_T macc_t;
__device__ __forceinline__ void fold_row(const RowAcc& A, float v, const float4 r1, const float4 r2,
                                         macc_t (&m)[8]) {
    const float fr = A.FR.x + A.FR.y, fg = A.FG.x + A.FG.y, fb = A.FB.x + A.FB.y;
    const macc_t w0 = (macc_t)fmaf(r1.w, fr, fmaf(r2.x, fg, r2.y * fb));
    const macc_t w1 = (macc_t)A.W1.x + (macc_t)A.W1.y, w2 = (macc_t)A.W2.x + (macc_t)A.W2.y;
    const macc_t vq = (macc_t)v;
    m[0] += fr; m[1] += fg; m[2] += fb;
    m[3] += w1;
    m[4] = fma(vq, w0, m[4]);
    m[5] += w2;
    m[6] = fma(vq, w1, m[6]);
    m[7] = fma(vq * vq, w0, m[7]);
}

__global__ void __launch_bounds__(BWD_THREADS) k_render_bwd(
    const ImgTable tab, const float4* __restrict__ rec, const int4* __restrict__ rects,
    const int* __restrict__ cell_start,
    const int* __restrict__ ext, const int* __restrict__ perm, const float* __restrict__ grad_out,
    double* __restrict__ moments, int ks, const float* __restrict__ img,
    const float* __restrict__ gt, float inv_numel) {
    __shared__ __align__(16) float4 gA[TILE_H][TILE_W / 2];
    // blue channel of two consecutive rows: gBB[r][cp] = {gb(r, 2cp), gb(r, 2cp+1), gb(r+1, 2cp),
    // gb(r+1, 2cp+1)} (row TILE_H = zeros), so a row pair reads its blue values with one LDS.128
    __shared__ __align__(16) float4 gBB[TILE_H][TILE_W / 2];
    __shared__ __align__(16) float2 gB[TILE_H + 1][TILE_W / 2];

    const int tile = blockIdx.x / ks;
    const int kpart = blockIdx.x % ks;    // split: this CTA takes every ks-th candidate group
    const int kimg = find_image_by_stile(tab, tile);
    const DevImg& im = tab.img[kimg];
    const int t = tile - im.stile_base;
    const int Tx0 = (t % im.ntx) * TILE_W;
    const int Ty0 = im.row_begin + (t / im.ntx) * TILE_H;
    const int Tx1 = min(Tx0 + TILE_W - 1, im.Ws - 1);
    const int Ty1 = min(Ty0 + TILE_H - 1, im.row_end - 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // stage dL/dI of the tile (zeros outside the image / band)
    for (int pp = threadIdx.x; pp < TILE_H * (TILE_W / 2); pp += BWD_THREADS) {
        int ry = pp / (TILE_W / 2), cp = pp % (TILE_W / 2);
#ifdef GSR_DIAG_BWD_NOSTAGE      // timing diagnostic only (wrong results): no dL/dI loads
        int y = Ty1 + 1, x = Tx0 + 2 * cp;
#else
        int y = Ty0 + ry, x = Tx0 + 2 * cp;
#endif
        float v[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        if (y <= Ty1) {
            const long long ro = im.out_off + ((long long)(y - im.row_begin) * im.Ws) * 3;
            const int nv = x + 1 <= Tx1 ? 6 : (x <= Tx1 ? 3 : 0);
            if (gt) {
                // fused L1 loss gradient (NEXT-1): dL/dI = sign(I - I_gt) / numel
                for (int k = 0; k < nv; ++k) {
                    const float d = img[ro + 3 * x + k] - gt[ro + 3 * x + k];
                    v[k] = d > 0.f ? inv_numel : (d < 0.f ? -inv_numel : 0.f);
                }
            } else if (im.io == 0) {
                const float* g = grad_out + ro;
                for (int k = 0; k < nv; ++k) v[k] = g[3 * x + k];
            } else {                           // NEXT-4 image formats (bf16 and/or planar CHW)
                for (int k = 0; k < nv; ++k)
                    v[k] = img_load(grad_out, im, img_index(im, y, x + k / 3, k % 3));
            }
        }
        gA[ry][cp] = make_float4(v[0], v[3], v[1], v[4]);
        gB[ry][cp] = make_float2(v[2], v[5]);
        if (ry == 0) gB[TILE_H][cp] = make_float2(0.f, 0.f);
    }
    __syncthreads();
    for (int pp = threadIdx.x; pp < TILE_H * (TILE_W / 2); pp += BWD_THREADS) {
        const int ry = pp / (TILE_W / 2), cp = pp % (TILE_W / 2);
        const float2 a = gB[ry][cp], b = gB[ry + 1][cp];
        gBB[ry][cp] = make_float4(a.x, a.y, b.x, b.y);
    }
    __syncthreads();

    const int cx_lo = (Tx0 - query_ext(ext, kimg, 0) + 1 + im.offx) / CELL;
    const int cx_hi = min(im.ncx - 1, (Tx1 + im.offx) / CELL);
    const int cy_lo = (Ty0 - im.row_begin - query_ext(ext, kimg, 1) + 1 + im.offy) / CELL;
    const int cy_hi = min(im.ncy - 1, (Ty1 - im.row_begin + im.offy) / CELL);
    const float invs = im.invsy;     // rows: dy = (y - ay)/sy - dl_y

    // Candidate compaction + grouping. Each warp scans its share of the tile's candidate spans
    // (32 records at a time, support-rect test only) and appends the candidates whose support
    // rect meets the tile to a per-warp queue in shared memory, with a key = the clipped column
    // range in TILE_W/KQ-px buckets (KQ x KQ keys). Every BWD_BATCH hits the warp
    // sorts its queue by key (stable counting sort) and evaluates groups of 32: every lane of a
    // group owns a Gaussian that touches the tile, and lanes with similar column ranges share a
    // group, so the union of their rects (the loop bounds) stays tight (C5: 52% -> ~67% of the
    // evaluated pairs inside some lane's support, tools/sim in DESIGN.md).
    constexpr int KQ = GSR_BWD_KQ;                // column buckets per axis
    constexpr int NB = KQ * KQ;                   // key buckets (x0 bucket, x1 bucket)
    constexpr int NBL = NB / 32;                  // buckets per lane in the scan
    constexpr int SCAN_U = GSR_BWD_SCAN_U;
    __shared__ int qp[BWD_WARPS][BWD_BATCH + 32 * SCAN_U];
    __shared__ unsigned short qk[BWD_WARPS][BWD_BATCH + 32 * SCAN_U];
    __shared__ int qs[BWD_WARPS][BWD_BATCH + 32 * SCAN_U];
    __shared__ int hist[BWD_WARPS][NB];
    const unsigned lt = (1u << lane) - 1u;
    int qn = 0;                                   // warp-uniform queue length
    auto group = [&](int p, bool act) {
        float4 r0 = make_float4(0.f, 0.f, 0.f, 0.f), r1 = r0, r2 = r0;
        int x0 = 1, x1 = 0, y0 = 1, y1 = 0;          // window rect (masks)
        int sx0 = 1, sx1 = 0, sy0 = 1, sy1 = 0;      // support rect (loop bounds)
        int gdst = 0;                                // the Gaussian's moment row (perm[p])
        if (act) {
            gdst = __ldg(perm + p);                  // issued early: used after the group loop
            r0 = __ldg(rec + (long long)REC_F4 * p);
            r1 = __ldg(rec + (long long)REC_F4 * p + 1);
            r2 = __ldg(rec + (long long)REC_F4 * p + 2);
            const int4 rc = __ldg(rects + p);
            unsigned xs = (unsigned)rc.z, ys = (unsigned)rc.w;
            x0 = (int)(xs & 0xffffu); x1 = (int)(xs >> 16);
            y0 = (int)(ys & 0xffffu); y1 = (int)(ys >> 16);
            xs = (unsigned)rc.x; ys = (unsigned)rc.y;
            sx0 = (int)(xs & 0xffffu); sx1 = (int)(xs >> 16);
            sy0 = (int)(ys & 0xffffu); sy1 = (int)(ys >> 16);
        }
        // warp-uniform loop bounds: union of the active support rects (rows and columns; pairs
        // outside a lane's support evaluate to exactly 0), and the column range inside every
        // active lane's window (no per-pixel x mask needed there)
        const int ya = max(Ty0, (int)__reduce_min_sync(0xffffffffu, act ? sy0 : 0x7fffffff));
        const int yb = min(Ty1, (int)__reduce_max_sync(0xffffffffu, act ? sy1 : -1));
        const int xa = max(Tx0, (int)__reduce_min_sync(0xffffffffu, act ? sx0 : 0x7fffffff));
        const int xb = min(Tx1, (int)__reduce_max_sync(0xffffffffu, act ? sx1 : -1));
        const int xia = (int)__reduce_max_sync(0xffffffffu, act ? x0 : -1);
        const int xib = (int)__reduce_min_sync(0xffffffffu, act ? x1 : 0x7fffffff);
        // column pairs relative to Tx0
        const int ca = (xa - Tx0) & ~1;
        const int ce = ((xb - Tx0) | 1) + 1;                  // exclusive, even
        int ma = ((xia - Tx0) + 1) & ~1;                      // first pair fully >= xia
        int mb = ((xib - Tx0) + 1) & ~1;                      // pairs [ma, mb) fully <= xib
        ma = min(max(ma, ca), ce);
        mb = min(max(mb, ma), ce);

        LaneG L;
        L.D2 = f2(r0.w);                                      // D = a1/s
        L.cr = f2(r1.w); L.cg = f2(r2.x); L.cb = f2(r2.y);
        L.x0 = x0; L.x1 = x1;
        const float kT = (float)Tx0 + r0.x;                    // Tx0 - ax
        const float tdl = r1.x;                                // -a1 dl_x
        macc_t m[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) m[k] = (macc_t)0;
#ifdef GSR_DIAG_BWD_NOEVAL       // timing diagnostic only (wrong results): no pair evaluation
        const int yb_ = r0.x == 12345.f ? yb : ya - 1;
        for (int y = ya; y <= yb_; y += 2) {
#else
        for (int y = ya; y <= yb; y += 2) {
#endif
            // rows y and y + 1 (the second one is a phantom when y == yb: u = -inf)
            const int y1r = y + 1;
            const bool has1 = y1r <= yb;
            const float dy0 = fmaf((float)y - r0.y, invs, -r0.z);
            const float dy1 = fmaf((float)y1r - r0.y, invs, -r0.z);
            const float v0 = r1.z * dy0, v1 = r1.z * dy1;
            const float u0 = (y >= y0 && y <= y1) ? -(v0 * v0) : -INFINITY;
            const float u1 = (has1 && y1r >= y0 && y1r <= y1) ? -(v1 * v1) : -INFINITY;
            const float2 T0 = f2(fmaf(r1.y, dy0, tdl)), T1 = f2(fmaf(r1.y, dy1, tdl));
            const float2 U0 = f2(u0), U1 = f2(u1);
            const int ry0 = y - Ty0, ry1 = has1 ? ry0 + 1 : ry0;
            const float4* gA0 = &gA[ry0][0];
            const float4* gA1 = &gA[ry1][0];
            const float4* gBr = &gBB[ry0][0];   // rows ry0, ry0 + 1 (a phantom row 1 has u = -inf)
            RowAcc A0, A1;
            A0.FR = A0.FG = A0.FB = A0.W1 = A0.W2 = f2(0.f);
            A1 = A0;
            row2_pairs<true>(ca, ma, gA0, gA1, gBr, kT, L, Tx0, T0, U0, T1, U1, A0, A1);
            row2_pairs<false>(ma, mb, gA0, gA1, gBr, kT, L, Tx0, T0, U0, T1, U1, A0, A1);
            row2_pairs<true>(mb, ce, gA0, gA1, gBr, kT, L, Tx0, T0, U0, T1, U1, A0, A1);
            fold_row(A0, v0, r1, r2, m);
            if (has1) fold_row(A1, v1, r1, r2, m);
        }
#ifndef GSR_BWD_NOATOM
        if (act) {
            double* dst = moments + 8LL * gdst;
#pragma unroll
            for (int k = 0; k < 8; ++k) atomicAdd(dst + k, (double)m[k]);
        }
#else   // diagnostic build only (wrong results): the cost of the atomics
        if (act && m[0] == 12345.f) moments[8LL * gdst] = m[1] + m[2] + m[3] + m[4] + m[5] + m[6] + m[7];
#endif
    };

    // sort the first cnt queue entries by key (stable: ranks via match_any in queue order),
    // evaluate them in groups of 32, then move the rest of the queue to the front
    auto flush = [&](int cnt) {
#ifdef GSR_DIAG_BWD_NOFLUSH      // timing diagnostic only (wrong results): scan without evaluation
        if (qk[warp][0] != 12345) { qn = 0; __syncwarp(); return; }
#endif
#pragma unroll
        for (int q = 0; q < NBL; ++q) hist[warp][NBL * lane + q] = 0;
        __syncwarp();
        for (int i0 = 0; i0 < cnt; i0 += 32) {
            const int i = i0 + lane;
            const bool v = i < cnt;
            const unsigned vm = __ballot_sync(0xffffffffu, v);
            if (v) {
                const int k = qk[warp][i];
                const unsigned peers = __match_any_sync(vm, k);
                if ((peers & lt) == 0) hist[warp][k] += __popc(peers);
            }
            __syncwarp();
        }
        {   // exclusive scan of the NB bucket counts (NBL consecutive buckets per lane)
            int h[NBL];
            int sum = 0;
#pragma unroll
            for (int q = 0; q < NBL; ++q) { h[q] = hist[warp][NBL * lane + q]; sum += h[q]; }
            int incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            __syncwarp();
            int run = incl - sum;
#pragma unroll
            for (int q = 0; q < NBL; ++q) { hist[warp][NBL * lane + q] = run; run += h[q]; }
            __syncwarp();
        }
        for (int i0 = 0; i0 < cnt; i0 += 32) {
            const int i = i0 + lane;
            const bool v = i < cnt;
            const unsigned vm = __ballot_sync(0xffffffffu, v);
            int k = 0, pos = 0;
            unsigned peers = 0;
            if (v) {
                k = qk[warp][i];
                peers = __match_any_sync(vm, k);
                pos = hist[warp][k] + __popc(peers & lt);
                qs[warp][pos] = qp[warp][i];
            }
            __syncwarp();
            if (v && (peers & lt) == 0) hist[warp][k] += __popc(peers);
            __syncwarp();
        }
        for (int g = 0; g < cnt; g += 32) {
            const bool act = g + lane < cnt;
            group(act ? qs[warp][g + lane] : 0, act);
        }
        const int rest = qn - cnt;                // < 32 * SCAN_U, moved to the front
        for (int r0 = 0; r0 < rest; r0 += 32) {
            int cp = 0;
            unsigned short ck = 0;
            const bool mv = r0 + lane < rest;
            if (mv) { cp = qp[warp][cnt + r0 + lane]; ck = qk[warp][cnt + r0 + lane]; }
            __syncwarp();
            if (mv) { qp[warp][r0 + lane] = cp; qk[warp][r0 + lane] = ck; }
            __syncwarp();
        }
        qn = rest;
        __syncwarp();
    };

#if GSR_BWD_CTASORT
    // CTA-wide rounds (GSR_BWD_CTASORT): every warp scans its share of the candidate chunks
    // into its own queue until it holds >= BWD_BATCH hits (or its share is exhausted); then the
    // CTA sorts the first <= BWD_BATCH hits of every warp's queue together -- key-major, then
    // warp order, then queue order (stable, deterministic) -- into one list of <= 4 BWD_BATCH
    // hits, and the warps evaluate its groups of 32 round-robin. The larger sorted batch makes
    // the groups' column ranges tighter (a replay of one C5 image: 86.6% instead of 81.3% of the
    // evaluated lane-pairs inside the lane's support) and the groups balance the warps.
    __shared__ int qs_cta[BWD_WARPS * BWD_BATCH];
    // [key][warp]: counts, then offsets (< 4 BWD_BATCH: 16 bits)
    __shared__ unsigned short hist_cta[NB * BWD_WARPS];
    __shared__ int sh_qn[BWD_WARPS], sh_done[BWD_WARPS], sh_tot[32];
    const int parts = ks * BWD_WARPS, part = kpart * BWD_WARPS + warp;
    int cy = cy_lo - 1, p0 = 0, s1 = 0;
    bool more = true;
    auto scan_step = [&]() {                          // one SCAN_U-chunk step of this warp
        while (p0 >= s1 && cy < cy_hi) {              // next non-empty cell row
            ++cy;
            const int row = im.cell_base + cy * im.ncx;
            const int s0 = cell_start[row + cx_lo];
            s1 = cell_start[row + cx_hi + 1];
            p0 = s0 + part * 32;
        }
        if (p0 >= s1) { more = false; return; }
        int4 rc[SCAN_U];
#pragma unroll
        for (int u = 0; u < SCAN_U; ++u) {
            const int p = p0 + u * parts * 32 + lane;
            rc[u] = p < s1 ? __ldg(rects + p) : make_int4(0, 0, 0x7fff7fff, 0);
        }
#pragma unroll
        for (int u = 0; u < SCAN_U; ++u) {
            const int p = p0 + u * parts * 32 + lane;
            bool hit = false;
            int key = 0;
            if (p < s1) {
                const unsigned xs = (unsigned)rc[u].x, ys = (unsigned)rc[u].y;
                const int x0 = (int)(xs & 0xffffu), x1 = (int)(xs >> 16);
                const int y0 = (int)(ys & 0xffffu), y1 = (int)(ys >> 16);
                hit = !(x1 < Tx0 || x0 > Tx1 || y1 < Ty0 || y0 > Ty1);
                key = ((max(x0, Tx0) - Tx0) / (TILE_W / KQ)) * KQ +
                      (min(x1, Tx1) - Tx0) / (TILE_W / KQ);
            }
            const unsigned hm = __ballot_sync(0xffffffffu, hit);
            if (hit) {
                const int slot = qn + __popc(hm & lt);
                qp[warp][slot] = p;
                qk[warp][slot] = (unsigned short)key;
            }
            qn += __popc(hm);
        }
        __syncwarp();
        p0 += parts * 32 * SCAN_U;
    };
    while (true) {
        while (more && qn < BWD_BATCH) scan_step();
        if (lane == 0) { sh_qn[warp] = qn; sh_done[warp] = more ? 0 : 1; }
        __syncthreads();
        int total = 0, mybase = 0, alldone = 1;
#pragma unroll
        for (int w = 0; w < BWD_WARPS; ++w) {
            const int c = min(sh_qn[w], BWD_BATCH);
            if (w < warp) mybase += c;
            total += c;
            alldone &= sh_done[w];
        }
        if (total == 0 && alldone) break;
        const int cnt = min(qn, BWD_BATCH);
        // counts per (key, warp)
        for (int k = lane; k < NB; k += 32) hist_cta[k * BWD_WARPS + warp] = 0;
        __syncwarp();
        for (int i0 = 0; i0 < cnt; i0 += 32) {
            const int i = i0 + lane;
            const bool v = i < cnt;
            const unsigned vm = __ballot_sync(0xffffffffu, v);
            if (v) {
                const int k = qk[warp][i];
                const unsigned peers = __match_any_sync(vm, k);
                if ((peers & lt) == 0) hist_cta[k * BWD_WARPS + warp] += __popc(peers);
            }
            __syncwarp();
        }
        __syncthreads();
        {   // exclusive scan of the NB x BWD_WARPS counts (key-major), one block scan
            constexpr int PER = NB * BWD_WARPS / BWD_THREADS;
            unsigned short* hseg = hist_cta + threadIdx.x * PER;
            int sum = 0;
#pragma unroll
            for (int q = 0; q < PER; ++q) sum += hseg[q];
            int incl = sum;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            if (lane == 31) sh_tot[warp] = incl;
            __syncthreads();
            int wbase = 0;
#pragma unroll
            for (int w = 0; w < BWD_WARPS; ++w) wbase += w < warp ? sh_tot[w] : 0;
            int run = wbase + incl - sum;
#pragma unroll
            for (int q = 0; q < PER; ++q) {
                const int t = hseg[q];
                hseg[q] = (unsigned short)run;
                run += t;
            }
        }
        __syncthreads();
        // stable scatter of this warp's first cnt hits
        for (int i0 = 0; i0 < cnt; i0 += 32) {
            const int i = i0 + lane;
            const bool v = i < cnt;
            const unsigned vm = __ballot_sync(0xffffffffu, v);
            int k = 0;
            unsigned peers = 0;
            if (v) {
                k = qk[warp][i];
                peers = __match_any_sync(vm, k);
                qs_cta[hist_cta[k * BWD_WARPS + warp] + __popc(peers & lt)] = qp[warp][i];
            }
            __syncwarp();
            if (v && (peers & lt) == 0) hist_cta[k * BWD_WARPS + warp] += __popc(peers);
            __syncwarp();
        }
        __syncthreads();
        for (int g = warp * 32; g < total; g += BWD_WARPS * 32) {
            const bool act = g + lane < total;
            group(act ? qs_cta[g + lane] : 0, act);
        }
        const int rest = qn - cnt;                    // < 32 * SCAN_U, moved to the front
        for (int r0 = 0; r0 < rest; r0 += 32) {
            int cp = 0;
            unsigned short ck = 0;
            const bool mv = r0 + lane < rest;
            if (mv) { cp = qp[warp][cnt + r0 + lane]; ck = qk[warp][cnt + r0 + lane]; }
            __syncwarp();
            if (mv) { qp[warp][r0 + lane] = cp; qk[warp][r0 + lane] = ck; }
            __syncwarp();
        }
        qn = rest;
        (void)mybase;
        __syncthreads();
    }
#else
    // Scan: SCAN_U chunks of 32 candidates (every parts-th chunk of the span, the same order as
    // one chunk at a time) have their rect loads in flight together, then are queued in order.
    for (int cy = cy_lo; cy <= cy_hi; ++cy) {
        const int row = im.cell_base + cy * im.ncx;
        const int s0 = cell_start[row + cx_lo], s1 = cell_start[row + cx_hi + 1];
        const int parts = ks * BWD_WARPS, part = kpart * BWD_WARPS + warp;
        for (int p0 = s0 + part * 32; p0 < s1; p0 += parts * 32 * SCAN_U) {
            int4 rc[SCAN_U];
#pragma unroll
            for (int u = 0; u < SCAN_U; ++u) {
                const int p = p0 + u * parts * 32 + lane;
                rc[u] = p < s1 ? __ldg(rects + p) : make_int4(0, 0, 0x7fff7fff, 0);
            }
#pragma unroll
            for (int u = 0; u < SCAN_U; ++u) {
                const int p = p0 + u * parts * 32 + lane;
                bool hit = false;
                int key = 0;
                if (p < s1) {
                    const unsigned xs = (unsigned)rc[u].x, ys = (unsigned)rc[u].y;
                    const int x0 = (int)(xs & 0xffffu), x1 = (int)(xs >> 16);
                    const int y0 = (int)(ys & 0xffffu), y1 = (int)(ys >> 16);
                    hit = !(x1 < Tx0 || x0 > Tx1 || y1 < Ty0 || y0 > Ty1);
                    key = ((max(x0, Tx0) - Tx0) / (TILE_W / KQ)) * KQ +
                          (min(x1, Tx1) - Tx0) / (TILE_W / KQ);
                }
                const unsigned hm = __ballot_sync(0xffffffffu, hit);
                if (hit) {
                    const int slot = qn + __popc(hm & lt);
                    qp[warp][slot] = p;
                    qk[warp][slot] = (unsigned short)key;
                }
                qn += __popc(hm);
            }
            __syncwarp();
            if (qn >= BWD_BATCH) flush(BWD_BATCH);
        }
    }
    if (qn > 0) flush(qn);
#endif
}

template <class T>
__global__ void k_finalize(const T* __restrict__ alpha, const T* __restrict__ mu,
                           const T* __restrict__ sigma, const T* __restrict__ rho,
                           const T* __restrict__ color, long long n,
                           const double* __restrict__ moments, float* __restrict__ d_alpha,
                           float* __restrict__ d_mu, float* __restrict__ d_sigma,
                           float* __restrict__ d_rho, float* __restrict__ d_color, RawParams raw,
                           int raw_mode, const int* __restrict__ gidx) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n) return;
    const long long i = gidx ? (long long)gidx[t] : t;      // subset mode: compact entry t
    float o[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (valid_at(alpha, mu, sigma, rho, color, i)) {
        const double* m = moments + 8 * t;
        double sx = ldf(sigma[2 * i]), sy = ldf(sigma[2 * i + 1]);
        double rh = ldf(rho[i]), al = ldf(alpha[i]);
        double c0 = ldf(color[3 * i]), c1 = ldf(color[3 * i + 1]), c2 = ldf(color[3 * i + 2]);
        double D = (1.0 - rh) * (1.0 + rh);
        double K = 1.0 / (TWO_PI * sx * sy * sqrt(D));
        double kp = sqrt(HALF_LOG2E / D), kv = sqrt(HALF_LOG2E);
        double cf = c0 * m[0] + c1 * m[1] + c2 * m[2];
        double S0 = al * K * cf;
        double Sp = m[3] / kp, Sv = m[4] / kv;
        double Spp = m[5] / (kp * kp), Spv = m[6] / (kp * kv), Svv = m[7] / HALF_LOG2E;
        double g9[9];
        g9[0] = K * cf;
        g9[1] = Sp / (sx * D);
        g9[2] = (Sv - rh * Sp / D) / sy;
        g9[3] = ((Spp + rh * Spv) / D - S0) / sx;
        g9[4] = (Svv - rh * Spv / D - S0) / sy;
        g9[5] = (rh * S0 + Spv - rh * Spp / D) / D;
        g9[6] = al * K * m[0];
        g9[7] = al * K * m[1];
        g9[8] = al * K * m[2];
        if (raw_mode) {
            // chain rule through the Gaussian Primary Head activations: sigmoid' from
            // the raw input in fp64 (exact also where the fp32 sigmoid saturates), tanh' likewise
            auto dsig = [](double r) { double e = exp(-fabs(r)); return e / ((1.0 + e) * (1.0 + e)); };
            auto dtanh = [](double r) { double t = tanh(r); return 1.0 - t * t; };
            g9[0] *= dsig((double)raw.raw_alpha[i]);
            g9[3] *= dsig((double)raw.raw_sigma[2 * i]);
            g9[4] *= dsig((double)raw.raw_sigma[2 * i + 1]);
            g9[5] *= (double)raw.rho_scale * dtanh((double)raw.raw_rho[i]);
            g9[6] *= dsig((double)raw.raw_color[3 * i]);
            g9[7] *= dsig((double)raw.raw_color[3 * i + 1]);
            g9[8] *= dsig((double)raw.raw_color[3 * i + 2]);
        }
        for (int k = 0; k < 9; ++k) o[k] = (float)g9[k];
    }
    d_alpha[t] = o[0];
    d_mu[2 * t] = o[1];
    d_mu[2 * t + 1] = o[2];
    d_sigma[2 * t] = o[3];
    d_sigma[2 * t + 1] = o[4];
    d_rho[t] = o[5];
    d_color[3 * t] = o[6];
    d_color[3 * t + 1] = o[7];
    d_color[3 * t + 2] = o[8];
}

}  // namespace

cudaError_t launch_render_bwd_moments(const ImgTable& tab, const Workspace& ws, const int* perm,
                                      const float* grad_out, double* moments, cudaStream_t st,
                                      const float* img, const float* gt, float inv_numel) {
    if (tab.total_tiles <= 0) return cudaSuccess;
    count_launches(1);
    int h = prof_begin(2, st);
    static std::atomic<int> slots_cache[64];       // per device (occupancy x SM count)
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
    int slots = slots_cache[dev].load(std::memory_order_relaxed);
    if (slots == 0) {
        slots = resident_slots(k_render_bwd, BWD_THREADS, 0);
        slots_cache[dev].store(slots, std::memory_order_relaxed);
    }
#ifdef GSR_FORCE_KS_BWD                 // A/B builds only
    const int ks = GSR_FORCE_KS_BWD;
#else
    const int ks = split_k_factor(tab.total_tiles, slots);
#endif
    k_render_bwd<<<tab.total_tiles * ks, BWD_THREADS, 0, st>>>(tab, ws.rec, ws.rects, ws.cell_start,
                                                               ws.ext,
                                                               perm, grad_out, moments, ks, img,
                                                               gt, inv_numel);
    prof_end(h, st);
    return cudaGetLastError();
}

cudaError_t launch_finalize(const void* alpha, const void* mu, const void* sigma,
                            const void* rho, const void* color, long long n,
                            const double* moments, float* d_alpha, float* d_mu, float* d_sigma,
                            float* d_rho, float* d_color, cudaStream_t st, const RawParams* raw,
                            bool params_bf16, const int* gidx) {
    if (n <= 0) return cudaSuccess;
    count_launches(1);
    int h = prof_begin(3, st);
    const unsigned grid = (unsigned)((n + 255) / 256);
    const RawParams rp = raw ? *raw : RawParams{};
    if (params_bf16) {
        using B = __nv_bfloat16;
        k_finalize<B><<<grid, 256, 0, st>>>((const B*)alpha, (const B*)mu, (const B*)sigma,
                                            (const B*)rho, (const B*)color, n, moments, d_alpha,
                                            d_mu, d_sigma, d_rho, d_color, rp, raw ? 1 : 0, gidx);
    } else {
        k_finalize<float><<<grid, 256, 0, st>>>((const float*)alpha, (const float*)mu,
                                                (const float*)sigma, (const float*)rho,
                                                (const float*)color, n, moments, d_alpha, d_mu,
                                                d_sigma, d_rho, d_color, rp, raw ? 1 : 0,
                                                gidx);
    }
    prof_end(h, st);
    return cudaGetLastError();
}

}  // namespace gsr
