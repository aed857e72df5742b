// render_fwd.cu -- K4: forward render (Eq. 4 / Alg. 1).
//
//   I[y][x][:] = sum over sorted records i with x0_i <= x <= x1_i, y0_i <= y <= y1_i of
//                c'_i * 2^(q_i(x,y)),  q = -(w^2 + v^2), w = a1 dx + b1 dy, v = c1 dy,
//                dx = (x - ax_i)/s - dl_x,  dy = (y - ay_i)/s - dl_y     (= x/s - mu_x, y/s - mu_y)
//
// Layout: one CTA per 32 x 32 HR tile, 4 warps side by side; warp w owns columns
// [Tx0 + 8w, Tx0 + 8w + 8) and lane l owns row Ty0 + l, i.e. every lane accumulates a 1 x 8
// pixel strip in registers. The x-window test is therefore warp-uniform per Gaussian (skip /
// full cover / partial), the y test is per lane and folded into the quadratic's constant term
// (u = -inf -> 2^q = 0). Candidate records (contiguous cell-row spans, binning.cu) are staged
// through shared memory by 1-D TMA bulk copies (cp.async.bulk + mbarrier, FWD_STAGES deep) and
// read as warp broadcasts. exp runs on the SFU (ex2.approx.ftz); the FP32 work is paired over
// neighbouring pixels with sm_100 FFMA2. Sums are two-level (per staged chunk, then total).
#include "gsr_internal.cuh"

namespace gsr {

namespace {

struct FwdProducer {
    int cy, cy_hi, row_stride, row0, cx_lo, cx_hi, cur, end;
    const int* cs;
    __device__ int next(int* start) {
        while (cur >= end) {
            if (++cy > cy_hi) return 0;
            int row = row0 + cy * row_stride;
            cur = cs[row + cx_lo];
            end = cs[row + cx_hi + 1];
        }
        int n = min(FWD_CHUNK, end - cur);
        *start = cur;
        cur += n;
        return n;
    }
};

__device__ __forceinline__ float2 f2(float a) { return make_float2(a, a); }

template <bool FULL>
__device__ __forceinline__ void fwd_gauss(const float4 r0, const float4 r1, const float4 r2,
                                          float yf, int y, float xw0f, int xw0, float invs,
                                          int x0, int x1, float2 (&pr)[4], float2 (&pg)[4],
                                          float2 (&pb)[4]) {
    unsigned ys = __float_as_uint(r2.w);
    int y0 = (int)(ys & 0xffffu), y1 = (int)(ys >> 16);
    float dy = fmaf(yf - r0.y, invs, -r0.w);
    float t = r1.y * dy;                 // b1 dy
    float v = r1.z * dy;                 // c1 dy
    float u = -(v * v);
    u = (y >= y0 && y <= y1) ? u : -INFINITY;
    const float kx0 = xw0f - r0.x;
    const float2 A2 = f2(r1.x), t2 = f2(t), u2 = f2(u), inv2 = f2(invs), ndl = f2(-r0.z);
    const float2 cr = f2(r1.w), cg = f2(r2.x), cb = f2(r2.y);
    const float2 k2 = f2(kx0);
#pragma unroll
    for (int jp = 0; jp < FWD_STRIP / 2; ++jp) {
        float2 kx = __fadd2_rn(k2, make_float2((float)(2 * jp), (float)(2 * jp + 1)));
        float2 dx = __ffma2_rn(kx, inv2, ndl);
        float2 w = __ffma2_rn(A2, dx, t2);                       // a1 dx + b1 dy
        float2 q = __ffma2_rn(make_float2(-w.x, -w.y), w, u2);   // -(w^2) - v^2
        if (!FULL) {
            int xa = xw0 + 2 * jp;
            q.x = (xa >= x0 && xa <= x1) ? q.x : -INFINITY;
            q.y = (xa + 1 >= x0 && xa + 1 <= x1) ? q.y : -INFINITY;
        }
        float2 e = make_float2(ex2_approx(q.x), ex2_approx(q.y));
        pr[jp] = __ffma2_rn(cr, e, pr[jp]);
        pg[jp] = __ffma2_rn(cg, e, pg[jp]);
        pb[jp] = __ffma2_rn(cb, e, pb[jp]);
    }
}

__global__ void __launch_bounds__(FWD_THREADS) k_render_fwd(const ImgTable tab,
                                                            const float4* __restrict__ rec,
                                                            const int* __restrict__ cell_start,
                                                            float* __restrict__ out) {
    __shared__ __align__(128) float4 srec[FWD_STAGES][FWD_CHUNK * 3];
    __shared__ __align__(8) uint64_t full_bar[FWD_STAGES];
    __shared__ int scount[FWD_STAGES];

    const int tile = blockIdx.x;
    const DevImg& im = tab.img[find_image_by_tile(tab, tile)];
    const int t = tile - im.tile_base;
    const int Tx0 = (t % im.ntx) * TILE_W;
    const int Ty0 = im.row_begin + (t / im.ntx) * TILE_H;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int xw0 = Tx0 + warp * FWD_STRIP;
    const int xwl = min(xw0 + FWD_STRIP - 1, im.Ws - 1);
    const int y = Ty0 + lane;
    const float yf = (float)y, xw0f = (float)xw0, invs = im.invs;

    FwdProducer prod;
    if (threadIdx.x == 0) {
        const int Tx1 = Tx0 + TILE_W - 1, Ty1 = Ty0 + TILE_H - 1;
        prod.cs = cell_start;
        prod.row0 = im.cell_base;
        prod.row_stride = im.ncx;
        prod.cx_lo = (Tx0 - im.wmax + 1 + im.offx) / CELL;
        prod.cx_hi = min(im.ncx - 1, (min(Tx1, im.Ws - 1) + im.offx) / CELL);
        prod.cy = (Ty0 - im.row_begin - im.hmax + 1 + im.offy) / CELL - 1;
        prod.cy_hi = min(im.ncy - 1, (min(Ty1, im.row_end - 1) - im.row_begin + im.offy) / CELL);
        prod.cur = prod.end = 0;
        for (int s = 0; s < FWD_STAGES; ++s) mbar_init(&full_bar[s], 1);
        fence_barrier_init();
    }
    __syncthreads();
    auto issue = [&](int s) {
        int start = 0;
        int n = prod.next(&start);
        scount[s] = n;
        if (n > 0) {
            uint32_t bytes = (uint32_t)n * 48u;
            mbar_arrive_expect_tx(&full_bar[s], bytes);
            tma_bulk_g2s(&srec[s][0], rec + 3LL * start, bytes, &full_bar[s]);
        } else {
            mbar_arrive(&full_bar[s]);
        }
    };
    if (threadIdx.x == 0)
        for (int s = 0; s < FWD_STAGES; ++s) issue(s);

    float2 tr[4], tg[4], tb[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) tr[j] = tg[j] = tb[j] = make_float2(0.f, 0.f);

    for (int k = 0;; ++k) {
        const int s = k % FWD_STAGES;
        mbar_wait(&full_bar[s], (uint32_t)((k / FWD_STAGES) & 1));
        const int n = scount[s];
        if (n == 0) break;
        float2 pr[4], pg[4], pb[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) pr[j] = pg[j] = pb[j] = make_float2(0.f, 0.f);
        const float4* sr = &srec[s][0];
        for (int g = 0; g < n; ++g) {
            const float4 r2 = sr[3 * g + 2];
            const unsigned xs = __float_as_uint(r2.z);
            const int x0 = (int)(xs & 0xffffu), x1 = (int)(xs >> 16);
            if (x1 < xw0 || x0 > xwl) continue;             // warp-uniform
            const float4 r0 = sr[3 * g], r1 = sr[3 * g + 1];
            if (x0 <= xw0 && x1 >= xwl)
                fwd_gauss<true>(r0, r1, r2, yf, y, xw0f, xw0, invs, x0, x1, pr, pg, pb);
            else
                fwd_gauss<false>(r0, r1, r2, yf, y, xw0f, xw0, invs, x0, x1, pr, pg, pb);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            tr[j] = __fadd2_rn(tr[j], pr[j]);
            tg[j] = __fadd2_rn(tg[j], pg[j]);
            tb[j] = __fadd2_rn(tb[j], pb[j]);
        }
        __syncthreads();                       // every warp is done with stage s
        if (threadIdx.x == 0) issue(s);        // refill it with chunk k + FWD_STAGES
    }

    if (y < im.row_end) {
        float* o = out + im.out_off + ((long long)(y - im.row_begin) * im.Ws) * 3;
#pragma unroll
        for (int j = 0; j < FWD_STRIP; ++j) {
            int x = xw0 + j;
            if (x < im.Ws) {
                float2 r = tr[j >> 1], g = tg[j >> 1], b = tb[j >> 1];
                o[3 * x + 0] = (j & 1) ? r.y : r.x;
                o[3 * x + 1] = (j & 1) ? g.y : g.x;
                o[3 * x + 2] = (j & 1) ? b.y : b.x;
            }
        }
    }
}

}  // namespace

cudaError_t launch_render_fwd(const ImgTable& tab, const Workspace& ws, float* out,
                              cudaStream_t st) {
    if (tab.total_tiles <= 0) return cudaSuccess;
    count_launches(1);
    int h = prof_begin(1, st);
    k_render_fwd<<<tab.total_tiles, FWD_THREADS, 0, st>>>(tab, ws.rec, ws.cell_start, out);
    prof_end(h, st);
    return cudaGetLastError();
}

}  // namespace gsr
