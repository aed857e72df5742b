// gsr_abi.cu -- the C-ABI of include/gsr.h: argument validation, per-image geometry (fp64,
// host), workspace carving and launch orchestration. No allocation, no stream sync.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/gsr.h"
#include "gsr_internal.cuh"

using namespace gsr;

// ---- launch accounting / phase profiler ----------------------------------------------------
namespace {
std::atomic<long long> g_launches{0};
struct Profiler {
    std::mutex mu;
    bool on = false;
    std::vector<cudaEvent_t> pool;
    struct Rec { int phase; cudaEvent_t a, b; };
    std::vector<Rec> open_, done;
    double ms[4] = {0, 0, 0, 0};
    long long calls[4] = {0, 0, 0, 0};
    cudaEvent_t get() {
        if (!pool.empty()) { cudaEvent_t e = pool.back(); pool.pop_back(); return e; }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
} g_prof;
}  // namespace

namespace {
// NVTX ranges around the phases' launches (GSR_NVTX=1, read once): binning (K1-K3),
// forward (K4), backward (K5), finalize (K6) -- host ranges around the enqueue, which nsys / ncu
// correlate with the kernels
bool nvtx_on() {
    static const bool on = [] {
        const char* e = std::getenv("GSR_NVTX");
        return e && e[0] && e[0] != '0';
    }();
    return on;
}
const char* const kPhaseName[4] = {"gsr:binning", "gsr:render_fwd", "gsr:render_bwd",
                                   "gsr:finalize"};
}  // namespace

namespace gsr {
void count_launches(long long k) { g_launches += k; }
int prof_begin(int phase, cudaStream_t st) {
    if (nvtx_on()) nvtxRangePushA(kPhaseName[phase & 3]);
    std::lock_guard<std::mutex> lk(g_prof.mu);
    if (!g_prof.on) return -1;
    Profiler::Rec r{phase, g_prof.get(), g_prof.get()};
    cudaEventRecord(r.a, st);
    g_prof.open_.push_back(r);
    return (int)g_prof.open_.size() - 1;
}
void prof_end(int handle, cudaStream_t st) {
    if (nvtx_on()) nvtxRangePop();
    if (handle < 0) return;
    std::lock_guard<std::mutex> lk(g_prof.mu);
    if (handle >= (int)g_prof.open_.size()) return;
    Profiler::Rec r = g_prof.open_[handle];
    cudaEventRecord(r.b, st);
    g_prof.done.push_back(r);
    g_prof.open_[handle].phase = -1;
    bool all_closed = true;
    for (auto& o : g_prof.open_) all_closed &= (o.phase < 0);
    if (all_closed) g_prof.open_.clear();
}
}  // namespace gsr

namespace {

constexpr int MAX_DIM = 65535;
#ifndef GSR_SCHED_DENSE
#define GSR_SCHED_DENSE 1
#endif

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

// Builds the per-image table; returns GSR_EINVAL on any host-checkable argument error.
gsr_status build_table(const gsr_image* imgs, int32_t n_imgs, int64_t n_total, double ratio,
                       ImgTable* tab, uint32_t flags = 0u) {
    if (!imgs || n_imgs < 1 || n_imgs > GSR_MAX_IMAGES) return GSR_EINVAL;
    if (n_total < 0 || n_total >= (1LL << 31)) return GSR_EINVAL;
    if (!std::isfinite(ratio) || !(ratio > 0.0) || ratio > 1.0) return GSR_EINVAL;
    std::memset(tab, 0, sizeof(*tab));
    tab->n_imgs = n_imgs;
    tab->params_bf16 = (flags & GSR_PARAMS_BF16) ? 1 : 0;
    const int io = ((flags & GSR_OUT_BF16) ? IO_BF16 : 0) | ((flags & GSR_OUT_CHW) ? IO_CHW : 0);
    // forward configuration: small tiles when every window is narrow
    double max_win = 0.0;
    for (int k = 0; k < n_imgs; ++k) {
        const gsr_image& g = imgs[k];
        const double gsy = g.scale_y > 0.0 ? g.scale_y : g.scale;
        double w = std::min(2.0 * ratio * g.scale * (double)g.lr_w, 2.0 * ratio * gsy * (double)g.lr_h);
        if (std::isfinite(w) && w > max_win) max_win = w;
    }
    tab->fwd_small = max_win < (double)FWD_SMALL_WINDOW ? 1 : 0;
    tab->ftile_w = tab->fwd_small ? FwdCfgSmall::TW : FwdCfgWide::TW;
    tab->ftile_h = tab->fwd_small ? FwdCfgSmall::TH : FwdCfgWide::TH;
    long long cells = 0, tiles = 0, ftiles = 0, prev_end = 0;
    for (int k = 0; k < n_imgs; ++k) {
        const gsr_image& g = imgs[k];
        if (g.lr_h < 1 || g.lr_w < 1) return GSR_EINVAL;
        if (!std::isfinite(g.scale) || !(g.scale >= 1.0)) return GSR_EINVAL;
        if (!std::isfinite(g.scale_y) || g.scale_y < 0.0 || (g.scale_y > 0.0 && g.scale_y < 1.0))
            return GSR_EINVAL;
        const double sx = g.scale, sy = g.scale_y > 0.0 ? g.scale_y : g.scale;   // reading R22
        if (g.g_off < prev_end || g.g_cnt < 0 || g.g_off + g.g_cnt > n_total) return GSR_EINVAL;
        if (g.out_off < 0) return GSR_EINVAL;
        prev_end = g.g_off + g.g_cnt;
        double hsd = std::floor(sy * (double)g.lr_h);   // readings R4, R22
        double wsd = std::floor(sx * (double)g.lr_w);
        if (hsd > MAX_DIM || wsd > MAX_DIM || hsd < 1 || wsd < 1) return GSR_EINVAL;
        DevImg& d = tab->img[k];
        d.sx = sx;
        d.sy = sy;
        d.hx = ratio * (double)g.lr_w;    // reading R1: x <-> W
        d.hy = ratio * (double)g.lr_h;
        d.g_off = g.g_off;
        d.g_cnt = g.g_cnt;
        d.out_off = g.out_off;
        d.invsx = (float)(1.0 / sx);
        d.invsy = (float)(1.0 / sy);
        d.H = g.lr_h; d.W = g.lr_w; d.Hs = (int)hsd; d.Ws = (int)wsd;
        int rb = g.row_begin, re = g.row_end < 0 ? d.Hs : g.row_end;
        if (rb < 0 || re > d.Hs || rb > re) return GSR_EINVAL;
        d.row_begin = rb; d.row_end = re;
        d.io = io;
        // bounds on the unclipped rect extent: width <= 2 s r W + 1 (+ fp64 rounding)
        d.wmax = (int)std::ceil(2.0 * sx * d.hx) + 2;
        d.hmax = (int)std::ceil(2.0 * sy * d.hy) + 2;
        d.offx = CELL * ceil_div(d.wmax, CELL);
        d.offy = CELL * ceil_div(d.hmax, CELL);
        int nrows = re - rb;
        if (nrows > 0) {
            d.ncx = (d.Ws - 1 + d.offx) / CELL + 1;
            d.ncy = (nrows - 1 + d.offy) / CELL + 1;
            d.ntx = ceil_div(d.Ws, TILE_W);
            d.nty = ceil_div(nrows, TILE_H);
            d.fntx = ceil_div(d.Ws, tab->ftile_w);
            d.fnty = ceil_div(nrows, tab->ftile_h);
        } else {
            d.ncx = d.ncy = d.ntx = d.nty = d.fntx = d.fnty = 0;
        }
        d.dense = (double)d.g_cnt * (CELL * CELL) >= 16.0 * (double)d.Ws * (double)d.Hs ? 1 : 0;
        d.cell_base = (int)cells;
        d.tile_base = (int)tiles;
        d.ftile_base = (int)ftiles;
        cells += (long long)d.ncx * d.ncy;
        tiles += (long long)d.ntx * d.nty;
        ftiles += (long long)d.fntx * d.fnty;
        if (cells >= (1LL << 30) || tiles >= (1LL << 30)) return GSR_EINVAL;
    }
    tab->total_cells = (int)cells;
    tab->total_tiles = (int)tiles;
    tab->total_ftiles = (int)ftiles;
    // launch order (GSR_SCHED_DENSE): densest images first -- a tile's cost grows with the
    // Gaussians per HR pixel (C2: 16 at s = 1, 1 at s = 4), so the heavy tiles start early and
    // the grid's tail holds light ones; results do not depend on the order
    for (int k = 0; k < n_imgs; ++k) tab->sched[k] = k;
#if GSR_SCHED_DENSE
    auto dens = [&](int k) {
        const DevImg& d = tab->img[k];
        return (double)d.g_cnt / std::max(1.0, (double)d.Hs * (double)d.Ws);
    };
    std::stable_sort(tab->sched, tab->sched + n_imgs,
                     [&](int a, int b) { return dens(a) > dens(b); });
#endif
    long long st = 0, sft = 0;
    for (int i = 0; i < n_imgs; ++i) {
        DevImg& d = tab->img[tab->sched[i]];
        d.stile_base = (int)st;
        d.sftile_base = (int)sft;
        st += (long long)d.ntx * d.nty;
        sft += (long long)d.fntx * d.fnty;
    }
    return GSR_OK;
}

gsr_image single(int64_t n, int32_t h, int32_t w, double s) {
    gsr_image g;
    g.lr_h = h; g.lr_w = w; g.scale = s; g.scale_y = 0.0;
    g.g_off = 0; g.g_cnt = n; g.out_off = 0; g.row_begin = 0; g.row_end = -1;
    return g;
}

bool params_ok(const void* a, const void* m, const void* s, const void* r, const void* c,
               int64_t n) {
    return n == 0 || (a && m && s && r && c);
}

size_t ws_bytes(const ImgTable& t, int64_t n) {
    return binning_bytes(n, t.total_cells, t.total_tiles);
}

gsr_status finish(cudaError_t e) {
    if (e != cudaSuccess) return GSR_ECUDA;
    return cudaGetLastError() == cudaSuccess ? GSR_OK : GSR_ECUDA;
}

struct Prepared {
    ImgTable tab;
    Workspace ws;
    int* perm = nullptr;
    uint32_t* keys = nullptr;
};

// gidx/m: subset mode (bin only the m Gaussians gidx[0..m), device int32, ascending, each owned
// by an image); gidx == nullptr: all n_total (m ignored)
gsr_status prepare(const void* alpha, const void* mu, const void* sigma, const void* rho,
                   const void* color, int64_t n_total, const gsr_image* imgs, int32_t n_imgs,
                   double ratio, void* workspace, size_t workspace_bytes, cudaStream_t st,
                   Prepared* P, bool bin, uint32_t flags = 0u, const int32_t* gidx = nullptr,
                   int64_t m = -1) {
    gsr_status s = build_table(imgs, n_imgs, n_total, ratio, &P->tab, flags);
    if (s != GSR_OK) return s;
    if (!params_ok(alpha, mu, sigma, rho, color, n_total)) return GSR_EINVAL;
    const int64_t nb = gidx ? m : n_total;
    if (gidx && (m < 0 || m > n_total)) return GSR_EINVAL;
    if (!workspace || workspace_bytes < ws_bytes(P->tab, nb)) return GSR_EWORKSPACE;
    carve_workspace(workspace, nb, P->tab.total_cells, P->tab.total_tiles, &P->ws);
    if (!bin) {
        binned_pointers(P->tab, nb, P->ws, &P->perm, &P->keys);
        return GSR_OK;
    }
    int h = prof_begin(0, st);
    cudaError_t e = bin_gaussians(alpha, mu, sigma, rho, color, nb, P->tab, P->ws, &P->perm,
                                  &P->keys, st, gidx);
    prof_end(h, st);
    return e == cudaSuccess ? GSR_OK : GSR_ECUDA;
}

}  // namespace

extern "C" {

#define GSR_STR2(x) #x
#define GSR_STR(x) GSR_STR2(x)
const char* gsr_version(void) {
    return "gsr-b200 0.4 (sm_100a; fwd 2x8 | 1x" GSR_STR(GSR_FWD_SMALL_STRIP) " px per lane, bwd tile 64x8, "
           "cell 16, support 13.5 sigma)";
}

gsr_status gsr_profile_enable(int32_t on) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    g_prof.on = on != 0;
    return GSR_OK;
}

gsr_status gsr_profile_collect(double* ms, int64_t* calls, int64_t* kernel_launches,
                               int32_t reset) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    for (auto& r : g_prof.done) {
        float t = 0.f;
        if (cudaEventSynchronize(r.b) != cudaSuccess) return GSR_ECUDA;
        cudaEventElapsedTime(&t, r.a, r.b);
        g_prof.ms[r.phase] += t;
        g_prof.calls[r.phase] += 1;
        g_prof.pool.push_back(r.a);
        g_prof.pool.push_back(r.b);
    }
    g_prof.done.clear();
    for (int k = 0; k < 4; ++k) {
        if (ms) ms[k] = g_prof.ms[k];
        if (calls) calls[k] = g_prof.calls[k];
    }
    if (kernel_launches) *kernel_launches = g_launches.load();
    if (reset) {
        for (int k = 0; k < 4; ++k) { g_prof.ms[k] = 0; g_prof.calls[k] = 0; }
        g_launches = 0;
    }
    return GSR_OK;
}

void gsr_tile_shape(int32_t* tile_w, int32_t* tile_h, int32_t* cell_w, int32_t* cell_h) {
    if (tile_w) *tile_w = TILE_W;
    if (tile_h) *tile_h = TILE_H;
    if (cell_w) *cell_w = CELL;
    if (cell_h) *cell_h = CELL;
}

gsr_status gsr_out_dims(int32_t lr_h, int32_t lr_w, double scale, int32_t* out_h,
                        int32_t* out_w) {
    if (lr_h < 1 || lr_w < 1 || !std::isfinite(scale) || !(scale >= 1.0)) return GSR_EINVAL;
    double h = std::floor(scale * (double)lr_h), w = std::floor(scale * (double)lr_w);
    if (h > MAX_DIM || w > MAX_DIM) return GSR_EINVAL;
    if (out_h) *out_h = (int32_t)h;
    if (out_w) *out_w = (int32_t)w;
    return GSR_OK;
}

gsr_status gsr_out_dims_v(int32_t lr_h, int32_t lr_w, double scale_x, double scale_y,
                          int32_t* out_h, int32_t* out_w) {
    if (lr_h < 1 || lr_w < 1 || !std::isfinite(scale_x) || !(scale_x >= 1.0)) return GSR_EINVAL;
    if (!std::isfinite(scale_y) || scale_y < 0.0 || (scale_y > 0.0 && scale_y < 1.0))
        return GSR_EINVAL;
    const double sy = scale_y > 0.0 ? scale_y : scale_x;              // reading R22
    double h = std::floor(sy * (double)lr_h), w = std::floor(scale_x * (double)lr_w);
    if (h > MAX_DIM || w > MAX_DIM) return GSR_EINVAL;
    if (out_h) *out_h = (int32_t)h;
    if (out_w) *out_w = (int32_t)w;
    return GSR_OK;
}

size_t gsr_workspace_bytes_batched(const gsr_image* imgs, int32_t n_imgs, int64_t n_total,
                                   double ratio) {
    ImgTable local;
    if (build_table(imgs, n_imgs, n_total, ratio, &local) != GSR_OK) return 0;
    return ws_bytes(local, n_total);
}

size_t gsr_workspace_bytes(int64_t n, int32_t lr_h, int32_t lr_w, double scale, double ratio) {
    gsr_image g = single(n, lr_h, lr_w, scale);
    return gsr_workspace_bytes_batched(&g, 1, n, ratio);
}

gsr_status gsr_render_fwd_batched_ex(const void* alpha, const void* mu, const void* sigma,
                                     const void* rho, const void* color, int64_t n_total,
                                     const gsr_image* imgs, int32_t n_imgs, double ratio,
                                     void* out, void* workspace, size_t workspace_bytes,
                                     uint32_t flags, void* stream) {
    if (!out) return GSR_EINVAL;
    if (flags & ~(GSR_OUT_BF16 | GSR_OUT_CHW | GSR_PARAMS_BF16)) return GSR_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    Prepared P;
    gsr_status s = prepare(alpha, mu, sigma, rho, color, n_total, imgs, n_imgs, ratio, workspace,
                           workspace_bytes, st, &P, true, flags);
    if (s != GSR_OK) return s;
    return finish(launch_render_fwd(P.tab, P.ws, (float*)out, st));
}

gsr_status gsr_render_fwd_batched(const float* alpha, const float* mu, const float* sigma,
                                  const float* rho, const float* color, int64_t n_total,
                                  const gsr_image* imgs, int32_t n_imgs, double ratio, float* out,
                                  void* workspace, size_t workspace_bytes, void* stream) {
    return gsr_render_fwd_batched_ex(alpha, mu, sigma, rho, color, n_total, imgs, n_imgs, ratio,
                                     out, workspace, workspace_bytes, 0u, stream);
}

gsr_status gsr_render_fwd(const float* alpha, const float* mu, const float* sigma,
                          const float* rho, const float* color, int64_t n, int32_t lr_h,
                          int32_t lr_w, double scale, double ratio, float* out, void* workspace,
                          size_t workspace_bytes, void* stream) {
    gsr_image g = single(n, lr_h, lr_w, scale);
    return gsr_render_fwd_batched(alpha, mu, sigma, rho, color, n, &g, 1, ratio, out, workspace,
                                  workspace_bytes, stream);
}

gsr_status gsr_render_bwd_moments_batched_ex(const void* alpha, const void* mu,
                                             const void* sigma, const void* rho,
                                             const void* color, int64_t n_total,
                                             const gsr_image* imgs, int32_t n_imgs, double ratio,
                                             const void* grad_out, double* moments,
                                             void* workspace, size_t workspace_bytes,
                                             uint32_t flags, void* stream) {
    if (!grad_out || (!moments && n_total > 0)) return GSR_EINVAL;
    if (flags & ~(GSR_REUSE_BINNING | GSR_OUT_BF16 | GSR_OUT_CHW | GSR_PARAMS_BF16))
        return GSR_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    Prepared P;
    gsr_status s = prepare(alpha, mu, sigma, rho, color, n_total, imgs, n_imgs, ratio, workspace,
                           workspace_bytes, st, &P, !(flags & GSR_REUSE_BINNING), flags);
    if (s != GSR_OK) return s;
    return finish(launch_render_bwd_moments(P.tab, P.ws, P.perm, (const float*)grad_out, moments,
                                            st));
}

gsr_status gsr_render_bwd_moments_batched(const float* alpha, const float* mu, const float* sigma,
                                          const float* rho, const float* color, int64_t n_total,
                                          const gsr_image* imgs, int32_t n_imgs, double ratio,
                                          const float* grad_out, double* moments, void* workspace,
                                          size_t workspace_bytes, void* stream) {
    return gsr_render_bwd_moments_batched_ex(alpha, mu, sigma, rho, color, n_total, imgs, n_imgs,
                                             ratio, grad_out, moments, workspace,
                                             workspace_bytes, 0u, stream);
}

gsr_status gsr_finalize_grads(const float* alpha, const float* mu, const float* sigma,
                              const float* rho, const float* color, int64_t n_total,
                              const double* moments, float* d_alpha, float* d_mu, float* d_sigma,
                              float* d_rho, float* d_color, void* stream) {
    return gsr_finalize_grads_ex(alpha, mu, sigma, rho, color, n_total, moments, d_alpha, d_mu,
                                 d_sigma, d_rho, d_color, 0u, stream);
}

gsr_status gsr_finalize_grads_ex(const void* alpha, const void* mu, const void* sigma,
                                 const void* rho, const void* color, int64_t n_total,
                                 const double* moments, float* d_alpha, float* d_mu,
                                 float* d_sigma, float* d_rho, float* d_color, uint32_t flags,
                                 void* stream) {
    if (n_total < 0 || (flags & ~GSR_PARAMS_BF16)) return GSR_EINVAL;
    if (n_total > 0 && (!params_ok(alpha, mu, sigma, rho, color, n_total) || !moments ||
                        !d_alpha || !d_mu || !d_sigma || !d_rho || !d_color))
        return GSR_EINVAL;
    return finish(launch_finalize(alpha, mu, sigma, rho, color, n_total, moments, d_alpha, d_mu,
                                  d_sigma, d_rho, d_color, (cudaStream_t)stream, nullptr,
                                  (flags & GSR_PARAMS_BF16) != 0));
}

// ---- subset (index-list) mode: one rank's halo of a row-band shard -------------------------
size_t gsr_workspace_bytes_subset(const gsr_image* imgs, int32_t n_imgs, int64_t n_total,
                                  int64_t m, double ratio) {
    ImgTable local;
    if (m < 0 || m > n_total) return 0;
    if (build_table(imgs, n_imgs, n_total, ratio, &local) != GSR_OK) return 0;
    return ws_bytes(local, m);
}

gsr_status gsr_render_fwd_subset(const void* alpha, const void* mu, const void* sigma,
                                 const void* rho, const void* color, int64_t n_total,
                                 const int32_t* idx, int64_t m, const gsr_image* imgs,
                                 int32_t n_imgs, double ratio, void* out, void* workspace,
                                 size_t workspace_bytes, uint32_t flags, void* stream) {
    if (!out || (!idx && m > 0)) return GSR_EINVAL;
    if (flags & ~(GSR_OUT_BF16 | GSR_OUT_CHW | GSR_PARAMS_BF16)) return GSR_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    Prepared P;
    static const int32_t dummy = 0;
    gsr_status s = prepare(alpha, mu, sigma, rho, color, n_total, imgs, n_imgs, ratio, workspace,
                           workspace_bytes, st, &P, true, flags, idx ? idx : &dummy, m);
    if (s != GSR_OK) return s;
    return finish(launch_render_fwd(P.tab, P.ws, (float*)out, st));
}

gsr_status gsr_render_bwd_moments_subset(const void* alpha, const void* mu, const void* sigma,
                                         const void* rho, const void* color, int64_t n_total,
                                         const int32_t* idx, int64_t m, const gsr_image* imgs,
                                         int32_t n_imgs, double ratio, const void* grad_out,
                                         double* moments, void* workspace,
                                         size_t workspace_bytes, uint32_t flags, void* stream) {
    if (!grad_out || (!moments && m > 0) || (!idx && m > 0)) return GSR_EINVAL;
    if (flags & ~(GSR_REUSE_BINNING | GSR_OUT_BF16 | GSR_OUT_CHW | GSR_PARAMS_BF16))
        return GSR_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    Prepared P;
    static const int32_t dummy = 0;
    gsr_status s = prepare(alpha, mu, sigma, rho, color, n_total, imgs, n_imgs, ratio, workspace,
                           workspace_bytes, st, &P, !(flags & GSR_REUSE_BINNING), flags,
                           idx ? idx : &dummy, m);
    if (s != GSR_OK) return s;
    return finish(launch_render_bwd_moments(P.tab, P.ws, P.perm, (const float*)grad_out, moments,
                                            st));
}

gsr_status gsr_finalize_grads_subset(const void* alpha, const void* mu, const void* sigma,
                                     const void* rho, const void* color, int64_t n_total,
                                     const int32_t* idx, int64_t m, const double* moments,
                                     float* d_alpha, float* d_mu, float* d_sigma, float* d_rho,
                                     float* d_color, uint32_t flags, void* stream) {
    if (n_total < 0 || m < 0 || m > n_total || (flags & ~GSR_PARAMS_BF16)) return GSR_EINVAL;
    if (m > 0 && (!idx || !params_ok(alpha, mu, sigma, rho, color, n_total) || !moments ||
                  !d_alpha || !d_mu || !d_sigma || !d_rho || !d_color))
        return GSR_EINVAL;
    return finish(launch_finalize(alpha, mu, sigma, rho, color, m, moments, d_alpha, d_mu,
                                  d_sigma, d_rho, d_color, (cudaStream_t)stream, nullptr,
                                  (flags & GSR_PARAMS_BF16) != 0, idx));
}

gsr_status gsr_render_bwd_batched_ex(const void* alpha, const void* mu, const void* sigma,
                                     const void* rho, const void* color, int64_t n_total,
                                     const gsr_image* imgs, int32_t n_imgs, double ratio,
                                     const void* grad_out, float* d_alpha, float* d_mu,
                                     float* d_sigma, float* d_rho, float* d_color,
                                     void* workspace, size_t workspace_bytes, uint32_t flags,
                                     void* stream) {
    if (!grad_out) return GSR_EINVAL;
    if (flags & ~(GSR_REUSE_BINNING | GSR_OUT_BF16 | GSR_OUT_CHW | GSR_PARAMS_BF16))
        return GSR_EINVAL;
    if (n_total > 0 && (!d_alpha || !d_mu || !d_sigma || !d_rho || !d_color)) return GSR_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    Prepared P;
    gsr_status s = prepare(alpha, mu, sigma, rho, color, n_total, imgs, n_imgs, ratio, workspace,
                           workspace_bytes, st, &P, !(flags & GSR_REUSE_BINNING), flags);
    if (s != GSR_OK) return s;
    if (n_total == 0) return GSR_OK;
    cudaMemsetAsync(P.ws.moments, 0, sizeof(double) * 8 * (size_t)n_total, st);
    cudaError_t e = launch_render_bwd_moments(P.tab, P.ws, P.perm, (const float*)grad_out,
                                              P.ws.moments, st);
    if (e != cudaSuccess) return GSR_ECUDA;
    return finish(launch_finalize(alpha, mu, sigma, rho, color, n_total, P.ws.moments, d_alpha,
                                  d_mu, d_sigma, d_rho, d_color, st, nullptr,
                                  P.tab.params_bf16 != 0));
}

gsr_status gsr_render_bwd_batched(const float* alpha, const float* mu, const float* sigma,
                                  const float* rho, const float* color, int64_t n_total,
                                  const gsr_image* imgs, int32_t n_imgs, double ratio,
                                  const float* grad_out, float* d_alpha, float* d_mu,
                                  float* d_sigma, float* d_rho, float* d_color, void* workspace,
                                  size_t workspace_bytes, void* stream) {
    return gsr_render_bwd_batched_ex(alpha, mu, sigma, rho, color, n_total, imgs, n_imgs, ratio,
                                     grad_out, d_alpha, d_mu, d_sigma, d_rho, d_color, workspace,
                                     workspace_bytes, 0u, stream);
}

gsr_status gsr_render_bwd(const float* alpha, const float* mu, const float* sigma,
                          const float* rho, const float* color, int64_t n, int32_t lr_h,
                          int32_t lr_w, double scale, double ratio, const float* grad_out,
                          float* d_alpha, float* d_mu, float* d_sigma, float* d_rho,
                          float* d_color, void* workspace, size_t workspace_bytes, void* stream) {
    gsr_image g = single(n, lr_h, lr_w, scale);
    return gsr_render_bwd_batched(alpha, mu, sigma, rho, color, n, &g, 1, ratio, grad_out,
                                  d_alpha, d_mu, d_sigma, d_rho, d_color, workspace,
                                  workspace_bytes, stream);
}

size_t gsr_train_workspace_bytes_batched(const gsr_image* imgs, int32_t n_imgs, int64_t n_total,
                                         double ratio) {
    size_t b = gsr_workspace_bytes_batched(imgs, n_imgs, n_total, ratio);
    if (b == 0) return 0;
    return b + (((size_t)n_total * 9 * sizeof(float) + 255) & ~(size_t)255) + 512;
}

gsr_status gsr_train_step_l1_batched(const float* raw_alpha, const float* offset, const float* ref,
                                     const float* raw_sigma, const float* raw_rho,
                                     const float* raw_color, int64_t n_total,
                                     const gsr_image* imgs, int32_t n_imgs, double ratio,
                                     float rho_scale, double inv_numel, const float* gt,
                                     float* out, double* loss, float* d_raw_alpha,
                                     float* d_offset, float* d_raw_sigma, float* d_raw_rho,
                                     float* d_raw_color, void* workspace, size_t workspace_bytes,
                                     void* stream) {
    if (!gt || !out || !loss) return GSR_EINVAL;
    if (!std::isfinite(rho_scale) || !(rho_scale > 0.f) || rho_scale > 1.f) return GSR_EINVAL;
    if (!std::isfinite(inv_numel)) return GSR_EINVAL;
    if (n_total > 0 && (!raw_alpha || !offset || !ref || !raw_sigma || !raw_rho || !raw_color ||
                        !d_raw_alpha || !d_offset || !d_raw_sigma || !d_raw_rho || !d_raw_color))
        return GSR_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    ImgTable tab;
    gsr_status s = build_table(imgs, n_imgs, n_total, ratio, &tab);
    if (s != GSR_OK) return s;
    const size_t act_bytes = (((size_t)n_total * 9 * sizeof(float) + 255) & ~(size_t)255);
    if (!workspace || workspace_bytes < gsr_train_workspace_bytes_batched(imgs, n_imgs, n_total,
                                                                          ratio))
        return GSR_EWORKSPACE;
    char* base = (char*)(((uintptr_t)workspace + 255) & ~uintptr_t(255));
    double* loss_acc = (double*)base;                    // 256 B slot
    float* act = (float*)(base + 256);
    float* a_alpha = act;
    float* a_mu = act + n_total;
    float* a_sigma = act + 3 * n_total;
    float* a_rho = act + 5 * n_total;
    float* a_color = act + 6 * n_total;
    void* rws = base + 256 + act_bytes;
    size_t rws_bytes = workspace_bytes - (size_t)((char*)rws - (char*)workspace);
    long long numel = 0;
    for (int k = 0; k < tab.n_imgs; ++k)
        numel += (long long)(tab.img[k].row_end - tab.img[k].row_begin) * tab.img[k].Ws * 3;
    const double inv = inv_numel > 0.0 ? inv_numel : (numel > 0 ? 1.0 / (double)numel : 0.0);

    cudaError_t e = launch_activate(raw_alpha, offset, ref, raw_sigma, raw_rho, raw_color,
                                    n_total, rho_scale, a_alpha, a_mu, a_sigma, a_rho, a_color, st);
    if (e != cudaSuccess) return GSR_ECUDA;
    Prepared P;
    s = prepare(a_alpha, a_mu, a_sigma, a_rho, a_color, n_total, imgs, n_imgs, ratio, rws,
                rws_bytes, st, &P, true);
    if (s != GSR_OK) return s;
    cudaMemsetAsync(loss_acc, 0, sizeof(double), st);
    e = launch_render_fwd(P.tab, P.ws, out, st, gt, loss_acc);
    if (e != cudaSuccess) return GSR_ECUDA;
    if (n_total > 0) {
        cudaMemsetAsync(P.ws.moments, 0, sizeof(double) * 8 * (size_t)n_total, st);
        e = launch_render_bwd_moments(P.tab, P.ws, P.perm, nullptr, P.ws.moments, st, out, gt,
                                      (float)inv);
        if (e != cudaSuccess) return GSR_ECUDA;
        RawParams raw{raw_alpha, raw_sigma, raw_rho, raw_color, rho_scale};
        e = launch_finalize(a_alpha, a_mu, a_sigma, a_rho, a_color, n_total, P.ws.moments,
                            d_raw_alpha, d_offset, d_raw_sigma, d_raw_rho, d_raw_color, st, &raw);
        if (e != cudaSuccess) return GSR_ECUDA;
    }
    e = launch_scale_loss(loss_acc, inv, st);
    if (e != cudaSuccess) return GSR_ECUDA;
    cudaMemcpyAsync(loss, loss_acc, sizeof(double), cudaMemcpyDeviceToDevice, st);
    return finish(cudaSuccess);
}

gsr_status gsr_pair_count_batched_ex(const void* alpha, const void* mu, const void* sigma,
                                     const void* rho, const void* color, int64_t n_total,
                                     const gsr_image* imgs, int32_t n_imgs, double ratio,
                                     uint32_t flags, int64_t* d_pairs, void* workspace,
                                     size_t workspace_bytes, void* stream) {
    if (!d_pairs || (flags & ~(GSR_SUPPORT | GSR_PARAMS_BF16))) return GSR_EINVAL;
    Prepared P;
    gsr_status s = prepare(alpha, mu, sigma, rho, color, n_total, imgs, n_imgs, ratio, workspace,
                           workspace_bytes, (cudaStream_t)stream, &P, false, flags);
    if (s != GSR_OK) return s;
    return finish(launch_pair_count(alpha, mu, sigma, rho, color, n_total, P.tab,
                                    (flags & GSR_SUPPORT) != 0, (long long*)d_pairs,
                                    (cudaStream_t)stream));
}

gsr_status gsr_pair_count_batched(const float* alpha, const float* mu, const float* sigma,
                                  const float* rho, const float* color, int64_t n_total,
                                  const gsr_image* imgs, int32_t n_imgs, double ratio,
                                  int64_t* d_pairs, void* workspace, size_t workspace_bytes,
                                  void* stream) {
    return gsr_pair_count_batched_ex(alpha, mu, sigma, rho, color, n_total, imgs, n_imgs, ratio,
                                     0u, d_pairs, workspace, workspace_bytes, stream);
}

gsr_status gsr_validate_params(const void* alpha, const void* mu, const void* sigma,
                               const void* rho, const void* color, int64_t n, uint32_t flags,
                               int64_t* result, void* stream) {
    if (n < 0 || !result || (flags & ~GSR_PARAMS_BF16)) return GSR_EINVAL;
    if (!params_ok(alpha, mu, sigma, rho, color, n)) return GSR_EINVAL;
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned long long init[2] = {0ull, ~0ull};
    cudaMemcpyAsync(result, init, sizeof(init), cudaMemcpyHostToDevice, st);
    return finish(launch_validate(alpha, mu, sigma, rho, color, n,
                                  (flags & GSR_PARAMS_BF16) != 0, (unsigned long long*)result,
                                  st));
}

// ---- K7 band planning (plan.cu) ----------------------------------------------------------
static gsr_status plan_prepare(const void* alpha, const void* mu, const void* sigma,
                               const void* rho, const void* color, int64_t n_total,
                               const gsr_image* imgs, int32_t n_imgs, double ratio,
                               uint32_t flags, uint32_t allowed, ImgTable* tab) {
    if (flags & ~allowed) return GSR_EINVAL;
    gsr_status s = build_table(imgs, n_imgs, n_total, ratio, tab, flags);
    if (s != GSR_OK) return s;
    if (!params_ok(alpha, mu, sigma, rho, color, n_total)) return GSR_EINVAL;
    return GSR_OK;
}

static void row_offsets(const ImgTable& tab, RowOff* ro) {
    std::memset(ro, 0, sizeof(*ro));
    for (int k = 0; k < tab.n_imgs; ++k)
        ro->off[k + 1] = ro->off[k] + (tab.img[k].row_end - tab.img[k].row_begin);
}

static gsr_status band_table(const ImgTable& tab, const int32_t* bounds, int32_t n_bands,
                             int32_t margin, BandTable* bt) {
    if (!bounds || n_bands < 1 || n_bands > MAX_BANDS || margin < 0) return GSR_EINVAL;
    std::memset(bt, 0, sizeof(*bt));
    bt->G = n_bands;
    bt->margin = margin;
    for (int k = 0; k < tab.n_imgs; ++k) {
        const int32_t* b = bounds + (size_t)k * (n_bands + 1);
        for (int g = 0; g <= n_bands; ++g) {
            if (b[g] < tab.img[k].row_begin || b[g] > tab.img[k].row_end) return GSR_EINVAL;
            if (g > 0 && b[g] < b[g - 1]) return GSR_EINVAL;
            bt->b[k][g] = b[g];
        }
    }
    return GSR_OK;
}

gsr_status gsr_row_pair_counts_batched(const void* alpha, const void* mu, const void* sigma,
                                       const void* rho, const void* color, int64_t n_total,
                                       const gsr_image* imgs, int32_t n_imgs, double ratio,
                                       uint32_t flags, int64_t* rowpairs, void* stream) {
    ImgTable tab;
    gsr_status s = plan_prepare(alpha, mu, sigma, rho, color, n_total, imgs, n_imgs, ratio, flags,
                                GSR_SUPPORT | GSR_PARAMS_BF16, &tab);
    if (s != GSR_OK) return s;
    if (!rowpairs) return GSR_EINVAL;
    RowOff ro;
    row_offsets(tab, &ro);
    return finish(launch_row_pair_counts(alpha, mu, sigma, rho, color, n_total, tab,
                                         (flags & GSR_SUPPORT) != 0, ro, (long long*)rowpairs,
                                         (cudaStream_t)stream));
}

gsr_status gsr_row_pair_counts_host(const void* alpha, const void* mu, const void* sigma,
                                    const void* rho, const void* color, int64_t n_total,
                                    const gsr_image* imgs, int32_t n_imgs, double ratio,
                                    uint32_t flags, int64_t* rowpairs) {
    ImgTable tab;
    gsr_status s = plan_prepare(alpha, mu, sigma, rho, color, n_total, imgs, n_imgs, ratio, flags,
                                GSR_SUPPORT | GSR_PARAMS_BF16, &tab);
    if (s != GSR_OK) return s;
    if (!rowpairs) return GSR_EINVAL;
    RowOff ro;
    row_offsets(tab, &ro);
    row_pair_counts_host(alpha, mu, sigma, rho, color, n_total, tab, (flags & GSR_SUPPORT) != 0,
                         ro, (long long*)rowpairs);
    return GSR_OK;
}

gsr_status gsr_band_span_batched(const void* alpha, const void* mu, const void* sigma,
                                 const void* rho, const void* color, int64_t n_total,
                                 const gsr_image* imgs, int32_t n_imgs, double ratio,
                                 uint32_t flags, const int32_t* bounds, int32_t n_bands,
                                 int32_t margin, int16_t* span, void* stream) {
    ImgTable tab;
    gsr_status s = plan_prepare(alpha, mu, sigma, rho, color, n_total, imgs, n_imgs, ratio, flags,
                                GSR_PARAMS_BF16, &tab);
    if (s != GSR_OK) return s;
    if (!span && n_total > 0) return GSR_EINVAL;
    std::vector<BandTable> bt(1);   // 16.6 KB: host heap, not the caller's stack
    s = band_table(tab, bounds, n_bands, margin, bt.data());
    if (s != GSR_OK) return s;
    return finish(launch_band_span(alpha, mu, sigma, rho, color, n_total, tab, bt[0], span,
                                   (cudaStream_t)stream));
}

size_t gsr_rank_halo_workspace_bytes(int64_t n_total) {
    return n_total < 0 ? 0 : rank_halo_bytes(n_total);
}

gsr_status gsr_rank_halo(const void* alpha, const void* mu, const void* sigma, const void* rho,
                         const void* color, int64_t n_total, const gsr_image* imgs,
                         int32_t n_imgs, double ratio, uint32_t flags, const int32_t* bounds,
                         int32_t n_bands, int32_t margin, int32_t rank, int32_t* idx,
                         int32_t* up, int32_t* down, int32_t* multi_pos, int32_t* multi_slot,
                         int64_t* totals, void* workspace, size_t workspace_bytes,
                         void* stream) {
    ImgTable tab;
    gsr_status s = plan_prepare(alpha, mu, sigma, rho, color, n_total, imgs, n_imgs, ratio, flags,
                                GSR_PARAMS_BF16, &tab);
    if (s != GSR_OK) return s;
    if (rank < 0 || rank >= n_bands || !totals) return GSR_EINVAL;
    if (n_total > 0 && (!idx || !up || !down || !multi_pos || !multi_slot)) return GSR_EINVAL;
    if (!workspace || workspace_bytes < rank_halo_bytes(n_total)) return GSR_EWORKSPACE;
    std::vector<BandTable> bt(1);
    s = band_table(tab, bounds, n_bands, margin, bt.data());
    if (s != GSR_OK) return s;
    return finish(launch_rank_halo(alpha, mu, sigma, rho, color, n_total, tab, bt[0], rank,
                                   workspace, idx, up, down, multi_pos, multi_slot,
                                   (long long*)totals, (cudaStream_t)stream));
}

gsr_status gsr_band_span_host(const void* alpha, const void* mu, const void* sigma,
                              const void* rho, const void* color, int64_t n_total,
                              const gsr_image* imgs, int32_t n_imgs, double ratio,
                              uint32_t flags, const int32_t* bounds, int32_t n_bands,
                              int32_t margin, int16_t* span) {
    ImgTable tab;
    gsr_status s = plan_prepare(alpha, mu, sigma, rho, color, n_total, imgs, n_imgs, ratio, flags,
                                GSR_PARAMS_BF16, &tab);
    if (s != GSR_OK) return s;
    if (!span && n_total > 0) return GSR_EINVAL;
    std::vector<BandTable> bt(1);
    s = band_table(tab, bounds, n_bands, margin, bt.data());
    if (s != GSR_OK) return s;
    band_span_host(alpha, mu, sigma, rho, color, n_total, tab, bt[0], span);
    return GSR_OK;
}

gsr_status gsr_debug_rects_ex(const float* alpha, const float* mu, const float* sigma,
                              const float* rho, const float* color, int64_t n, int32_t lr_h,
                              int32_t lr_w, double scale, double ratio, uint32_t flags,
                              int32_t* rects, void* stream) {
    if (flags & ~GSR_SUPPORT) return GSR_EINVAL;
    gsr_image g = single(n, lr_h, lr_w, scale);
    ImgTable tab;
    gsr_status s = build_table(&g, 1, n, ratio, &tab);
    if (s != GSR_OK) return s;
    if (!params_ok(alpha, mu, sigma, rho, color, n) || (n > 0 && !rects)) return GSR_EINVAL;
    return finish(launch_debug_rects(alpha, mu, sigma, rho, color, n, tab,
                                     (flags & GSR_SUPPORT) != 0, rects, (cudaStream_t)stream));
}

gsr_status gsr_debug_rects(const float* alpha, const float* mu, const float* sigma,
                           const float* rho, const float* color, int64_t n, int32_t lr_h,
                           int32_t lr_w, double scale, double ratio, int32_t* rects,
                           void* stream) {
    return gsr_debug_rects_ex(alpha, mu, sigma, rho, color, n, lr_h, lr_w, scale, ratio, 0u,
                              rects, stream);
}

gsr_status gsr_debug_tile_lists(const float* alpha, const float* mu, const float* sigma,
                                const float* rho, const float* color, int64_t n, int32_t lr_h,
                                int32_t lr_w, double scale, double ratio, int32_t* counts,
                                int32_t* ids, int32_t* cells, void* workspace,
                                size_t workspace_bytes, void* stream) {
    if (!counts && !ids) return GSR_EINVAL;
    if (ids && !cells) return GSR_EINVAL;
    gsr_image g = single(n, lr_h, lr_w, scale);
    cudaStream_t st = (cudaStream_t)stream;
    Prepared P;
    gsr_status s = prepare(alpha, mu, sigma, rho, color, n, &g, 1, ratio, workspace,
                           workspace_bytes, st, &P, true);
    if (s != GSR_OK) return s;
    return finish(launch_debug_tile_lists(P.tab, P.ws, P.perm, P.keys, counts, ids, cells, st));
}

gsr_status gsr_debug_fwd_tile_lists(const float* alpha, const float* mu, const float* sigma,
                                    const float* rho, const float* color, int64_t n,
                                    int32_t lr_h, int32_t lr_w, double scale, double ratio,
                                    int32_t* geom, const int32_t* offsets, int32_t* counts,
                                    int32_t* ids, uint8_t* paths, void* workspace,
                                    size_t workspace_bytes, void* stream) {
    if (!geom || (!offsets && !counts) || (offsets && (!ids || !paths))) return GSR_EINVAL;
    gsr_image g = single(n, lr_h, lr_w, scale);
    cudaStream_t st = (cudaStream_t)stream;
    Prepared P;
    gsr_status s = prepare(alpha, mu, sigma, rho, color, n, &g, 1, ratio, workspace,
                           workspace_bytes, st, &P, true);
    if (s != GSR_OK) return s;
    geom[0] = P.tab.ftile_w;
    geom[1] = P.tab.ftile_h;
    geom[2] = P.tab.total_ftiles;
    return finish(launch_debug_fwd_lists(P.tab, P.ws, P.perm, offsets, counts, ids, paths, st));
}

}  // extern "C"
