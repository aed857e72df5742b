/*
 * abi_check.c -- TEST: drives libgsr.so through its C-ABI (include/gsr.h) from plain C, with no
 * Python or PyTorch in the process. CPU part (always): version, output sizes (R4, R22),
 * workspace sizes and host-checkable errors. GPU part (argv[1] == "gpu"): renders a small
 * seeded scene with gsr_render_fwd / gsr_render_bwd on device buffers (cudaMalloc) and compares
 * with the float64 oracle (oracle/gsr_oracle.c, linked into this test only) under the parity
 * gates of tests/_util.py (forward max-abs 1e-5; backward 1e-4 of the largest gradient per
 * field, a looser form of the Python gate that needs no term masses).
 * Exit code 0 = pass.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/gsr.h"

/* the oracle's entry points (oracle/gsr_oracle.c) */
void gsr_oracle_out_dims(int H, int W, double sw, double sh, int* Hs, int* Ws);
int gsr_oracle_render_fwd(int64_t n, const double* alpha, const double* mu, const double* sigma,
                          const double* rho, const double* color, int H, int W, double sw,
                          double sh, double r, int mode, int row_begin, int row_end, double* out);
int gsr_oracle_render_bwd(int64_t n, const double* alpha, const double* mu, const double* sigma,
                          const double* rho, const double* color, int H, int W, double sw,
                          double sh, double r, int mode, int row_begin, int row_end,
                          const double* grad_out, int64_t nidx, const int64_t* idx,
                          double* d_alpha, double* d_mu, double* d_sigma, double* d_rho,
                          double* d_color, double* absmass, double* termabs);

/* CUDA runtime (libcudart), declared here so the test needs no CUDA headers */
int cudaMalloc(void** p, size_t n);
int cudaFree(void* p);
int cudaMemcpy(void* dst, const void* src, size_t n, int kind);
int cudaDeviceSynchronize(void);
#define H2D 1
#define D2H 2

static int fails = 0;
#define CHECK(c, ...) do { if (!(c)) { printf("FAIL %s:%d: ", __FILE__, __LINE__); \
    printf(__VA_ARGS__); printf("\n"); ++fails; } } while (0)

/* a small deterministic generator (no method arithmetic): xorshift64* -> U[0,1) */
static uint64_t rs = 88172645463325252ull;
static double urand(void) {
    rs ^= rs >> 12; rs ^= rs << 25; rs ^= rs >> 27;
    return (double)((rs * 2685821657736338717ull) >> 11) * (1.0 / 9007199254740992.0);
}

static int cpu_part(void) {
    printf("%s\n", gsr_version());
    int32_t h = 0, w = 0;
    CHECK(gsr_out_dims(48, 48, 4.0, &h, &w) == GSR_OK && h == 192 && w == 192, "dims x4");
    CHECK(gsr_out_dims(339, 510, 4.0, &h, &w) == GSR_OK && h == 1356 && w == 2040, "dims C3");
    CHECK(gsr_out_dims(10, 10, 0.5, &h, &w) == GSR_EINVAL, "s < 1 rejected");
    CHECK(gsr_workspace_bytes(1000, 16, 16, 4.0, 0.1) > 0, "workspace bytes");
    gsr_image im;
    memset(&im, 0, sizeof im);
    im.lr_h = 10; im.lr_w = 12; im.scale = 3.0; im.scale_y = 2.0; im.g_cnt = 5; im.row_end = -1;
    CHECK(gsr_workspace_bytes_batched(&im, 1, 5, 0.1) > 0, "scale vector accepted");
    im.scale_y = 0.5;
    CHECK(gsr_workspace_bytes_batched(&im, 1, 5, 0.1) == 0, "scale_y < 1 rejected");
    float dummy[4];
    CHECK(gsr_render_fwd(dummy, dummy, dummy, dummy, dummy, 10, 4, 4, 2.0, 0.0, dummy, dummy,
                         1u << 30, NULL) == GSR_EINVAL, "ratio 0 rejected");
    CHECK(gsr_render_fwd(dummy, dummy, dummy, dummy, dummy, 10, 4, 4, 2.0, 0.1, dummy, dummy, 16,
                         NULL) == GSR_EWORKSPACE, "small workspace rejected");
    return fails;
}

static int gpu_part(void) {
    const int H = 12, W = 14, m = 4;
    const double s = 3.5, r = 0.1;
    const int64_t n = (int64_t)m * H * W;
    int32_t Hs, Ws;
    gsr_out_dims(H, W, s, &Hs, &Ws);
    const size_t npx = (size_t)Hs * Ws * 3;
    float *a = malloc(4 * n), *mu = malloc(8 * n), *sg = malloc(8 * n), *rh = malloc(4 * n),
          *c = malloc(12 * n), *img = malloc(4 * npx), *g = malloc(4 * npx);
    double *ad = malloc(8 * n), *mud = malloc(16 * n), *sgd = malloc(16 * n),
           *rhd = malloc(8 * n), *cd = malloc(24 * n), *ref = malloc(8 * npx),
           *gd = malloc(8 * npx);
    int64_t i = 0;
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x)
            for (int k = 0; k < m; ++k, ++i) {       /* image-like recipe, float32 values */
                a[i] = (float)(0.02 + 0.2 * urand());
                mu[2 * i] = (float)(x + urand()); mu[2 * i + 1] = (float)(y + urand());
                sg[2 * i] = (float)(0.15 + 0.5 * urand()); sg[2 * i + 1] = (float)(0.15 + 0.5 * urand());
                rh[i] = (float)(1.6 * urand() - 0.8);
                for (int q = 0; q < 3; ++q) c[3 * i + q] = (float)urand();
            }
    for (size_t p = 0; p < npx; ++p) g[p] = (float)(2.0 * urand() - 1.0);
    for (i = 0; i < n; ++i) {
        ad[i] = a[i]; rhd[i] = rh[i];
        for (int q = 0; q < 2; ++q) { mud[2 * i + q] = mu[2 * i + q]; sgd[2 * i + q] = sg[2 * i + q]; }
        for (int q = 0; q < 3; ++q) cd[3 * i + q] = c[3 * i + q];
    }
    for (size_t p = 0; p < npx; ++p) gd[p] = g[p];

    void *da, *dmu, *dsg, *drh, *dc, *dimg, *dg, *ws, *ga, *gmu, *gsg, *grh, *gc;
    size_t wsb = gsr_workspace_bytes(n, H, W, s, r);
    cudaMalloc(&da, 4 * n); cudaMalloc(&dmu, 8 * n); cudaMalloc(&dsg, 8 * n);
    cudaMalloc(&drh, 4 * n); cudaMalloc(&dc, 12 * n); cudaMalloc(&dimg, 4 * npx);
    cudaMalloc(&dg, 4 * npx); cudaMalloc(&ws, wsb);
    cudaMalloc(&ga, 4 * n); cudaMalloc(&gmu, 8 * n); cudaMalloc(&gsg, 8 * n);
    cudaMalloc(&grh, 4 * n); cudaMalloc(&gc, 12 * n);
    cudaMemcpy(da, a, 4 * n, H2D); cudaMemcpy(dmu, mu, 8 * n, H2D); cudaMemcpy(dsg, sg, 8 * n, H2D);
    cudaMemcpy(drh, rh, 4 * n, H2D); cudaMemcpy(dc, c, 12 * n, H2D); cudaMemcpy(dg, g, 4 * npx, H2D);

    CHECK(gsr_render_fwd(da, dmu, dsg, drh, dc, n, H, W, s, r, dimg, ws, wsb, NULL) == GSR_OK,
          "gsr_render_fwd");
    CHECK(gsr_render_bwd(da, dmu, dsg, drh, dc, n, H, W, s, r, dg, ga, gmu, gsg, grh, gc, ws, wsb,
                         NULL) == GSR_OK, "gsr_render_bwd");
    cudaDeviceSynchronize();
    cudaMemcpy(img, dimg, 4 * npx, D2H);
    gsr_oracle_render_fwd(n, ad, mud, sgd, rhd, cd, H, W, s, s, r, 1, 0, Hs, ref);
    double err = 0.0;
    for (size_t p = 0; p < npx; ++p) err = fmax(err, fabs((double)img[p] - ref[p]));
    printf("forward max-abs error %.3e\n", err);
    CHECK(err <= 1e-5, "forward parity %.3e", err);

    double *oa = malloc(8 * n), *om = malloc(16 * n), *os = malloc(16 * n), *orh = malloc(8 * n),
           *oc = malloc(24 * n);
    gsr_oracle_render_bwd(n, ad, mud, sgd, rhd, cd, H, W, s, s, r, 1, 0, Hs, gd, 0, NULL, oa, om,
                          os, orh, oc, NULL, NULL);
    float *fa = malloc(4 * n), *fm = malloc(8 * n), *fs = malloc(8 * n), *fr = malloc(4 * n),
          *fc = malloc(12 * n);
    cudaMemcpy(fa, ga, 4 * n, D2H); cudaMemcpy(fm, gmu, 8 * n, D2H); cudaMemcpy(fs, gsg, 8 * n, D2H);
    cudaMemcpy(fr, grh, 4 * n, D2H); cudaMemcpy(fc, gc, 12 * n, D2H);
    const struct { const char* name; const float* got; const double* want; int64_t len; } F[5] = {
        {"alpha", fa, oa, n}, {"mu", fm, om, 2 * n}, {"sigma", fs, os, 2 * n},
        {"rho", fr, orh, n}, {"color", fc, oc, 3 * n}};
    for (int f = 0; f < 5; ++f) {
        double mx = 0.0, e = 0.0;
        for (int64_t j = 0; j < F[f].len; ++j) mx = fmax(mx, fabs(F[f].want[j]));
        for (int64_t j = 0; j < F[f].len; ++j) e = fmax(e, fabs((double)F[f].got[j] - F[f].want[j]));
        printf("d_%s relative error %.3e\n", F[f].name, e / mx);
        CHECK(e <= 1e-4 * mx, "d_%s parity %.3e", F[f].name, e / mx);
    }
    return fails;
}

int main(int argc, char** argv) {
    cpu_part();
    if (argc > 1 && strcmp(argv[1], "gpu") == 0) gpu_part();
    printf(fails ? "abi_check: %d failure(s)\n" : "abi_check: ok\n", fails);
    return fails ? 1 : 0;
}
