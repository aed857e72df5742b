// Pipe-throughput microbenchmarks for the roofline denominators (SFU ex2, FP32 FFMA/FFMA2).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
// Each kernel runs ITERS iterations of UNROLL independent chains per thread. Every CTA records
// its SM id and clock64() at the start and end of the loop; per SM the busy span is
// max(end) - min(start) over the CTAs that ran there (clock64 is a per-SM counter), so the rate
// counts exactly the work that SM did, whether or not all its CTAs were co-resident.
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096

__device__ __forceinline__ void rec3(long long* cyc, long long t0, long long t1) {
  unsigned smid; asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  cyc[3 * blockIdx.x] = smid; cyc[3 * blockIdx.x + 1] = t0; cyc[3 * blockIdx.x + 2] = t1;
}

__device__ __forceinline__ float ex2f(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

__global__ void k_ex2(float* out, long long* cyc, float seed) {
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = seed * (threadIdx.x + j) * 1e-9f - 0.5f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = ex2f(a[j]) - 1.0f;   // ex2 + FADD per element
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int j = 0; j < 8; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) rec3(cyc, t0, t1);
}

__global__ void k_ex2_pure(float* out, long long* cyc, float seed) {
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = seed * (threadIdx.x + j) * 1e-9f - 0.5f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = ex2f(a[j]);   // chained ex2 (value converges to ~0.64)
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int j = 0; j < 8; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) rec3(cyc, t0, t1);
}

__global__ void k_ffma(float* out, long long* cyc, float seed) {
  float a[8], b = seed * 1e-7f + 0.999f, c = seed * 1e-8f;
  float b2 = b * 0.5f, c2 = c + 1.0f;
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x + j;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) { a[j] = fmaf(a[j], b, c); a[j] = fmaf(a[j], b2, c2); }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int j = 0; j < 8; ++j) s += a[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) rec3(cyc, t0, t1);
}

__global__ void k_ffma2(float* out, long long* cyc, float seed) {
  float2 a[8], b = make_float2(seed * 1e-7f + 0.999f, 0.998f), c = make_float2(seed * 1e-8f, 1e-3f);
  float2 b2 = make_float2(0.5f, 0.25f), c2 = make_float2(1.0f, 2.0f);
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = make_float2(threadIdx.x + j, j);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) { a[j] = __ffma2_rn(a[j], b, c); a[j] = __ffma2_rn(a[j], b2, c2); }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int j = 0; j < 8; ++j) s += a[j].x + a[j].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) rec3(cyc, t0, t1);
}

// FFMA2 with three distinct register pairs per instruction (no operand reuse between
// consecutive instructions): exposes register-file bank limits on the paired FMA path
__global__ void k_ffma2_norreuse(float* out, long long* cyc, float seed) {
  float2 a[8], x[8], y[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    a[j] = make_float2(threadIdx.x + j, j);
    x[j] = make_float2(0.999f + j * 1e-4f + seed * 1e-9f + threadIdx.x * 1e-10f, 0.998f - j * 1e-4f);
    y[j] = make_float2(1e-3f * j + threadIdx.x * 1e-10f, 2e-3f * j + seed * 1e-9f);
  }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = __ffma2_rn(x[j], a[j], y[(j + 3) & 7]);
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = __ffma2_rn(y[j], a[j], x[(j + 5) & 7]);
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int j = 0; j < 8; ++j) s += a[j].x + a[j].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) rec3(cyc, t0, t1);
}

// forward-like mix per element: 2 FFMA (q), 1 MUFU, 3 FFMA (rgb accumulate)
__global__ void k_mix(float* out, long long* cyc, float seed) {
  float d[8], ar[8], ag[8], ab[8];
  float A = -0.7f, t = seed * 1e-9f, u = -0.1f, cr = 0.3f, cg = 0.2f, cb = 0.1f;
#pragma unroll
  for (int j = 0; j < 8; ++j) { d[j] = (threadIdx.x & 7) * 0.01f + j * 0.125f; ar[j] = ag[j] = ab[j] = 0.f; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float q = fmaf(fmaf(A, d[j], t), d[j], u);
      float e = ex2f(q);
      ar[j] = fmaf(cr, e, ar[j]); ag[j] = fmaf(cg, e, ag[j]); ab[j] = fmaf(cb, e, ab[j]);
    }
    t += 1e-7f;
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0; for (int j = 0; j < 8; ++j) s += ar[j] + ag[j] + ab[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) rec3(cyc, t0, t1);
}

// accuracy of ex2.approx.ftz.f32 (MUFU.EX2) against exp2 in fp64, over x in [lo, hi]
__global__ void k_ex2_acc(double lo, double hi, long long n, double* worst) {
  double w = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    float x = (float)(lo + (hi - lo) * (double)i / (double)n);
    double ref = exp2((double)x);
    double rel = fabs((double)ex2f(x) - ref) / ref;
    w = rel > w ? rel : w;
  }
  for (int o = 16; o > 0; o >>= 1) { double t = __shfl_xor_sync(0xffffffffu, w, o); w = t > w ? t : w; }
  if ((threadIdx.x & 31) == 0) atomicMax((unsigned long long*)worst, __double_as_longlong(w));
}

typedef void (*kfn)(float*, long long*, float);

static void run(const char* name, kfn k, double ops_per_elem_iter, int threads, int blocks_per_sm) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int blocks = sms * blocks_per_sm;
  float* out; long long* cyc;
  cudaMalloc(&out, sizeof(float) * blocks * threads);
  cudaMalloc(&cyc, 3 * sizeof(long long) * blocks);
  k<<<blocks, threads>>>(out, cyc, 1.0f);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<blocks, threads>>>(out, cyc, 2.0f);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  long long* h = new long long[3 * blocks];
  cudaMemcpy(h, cyc, 3 * sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  // per SM: CTAs it ran, busy span = max(end) - min(start)
  long long* lo = new long long[1024]; long long* hi = new long long[1024]; int* cnt = new int[1024];
  for (int i = 0; i < 1024; ++i) { lo[i] = 0x7fffffffffffffffLL; hi[i] = 0; cnt[i] = 0; }
  for (int b = 0; b < blocks; ++b) {
    int sm = (int)h[3 * b];
    if (h[3 * b + 1] < lo[sm]) lo[sm] = h[3 * b + 1];
    if (h[3 * b + 2] > hi[sm]) hi[sm] = h[3 * b + 2];
    cnt[sm]++;
  }
  double rmin = 1e30, rmax = 0, rsum = 0; int nsm = 0; long long span_max = 0;
  for (int i = 0; i < 1024; ++i) {
    if (!cnt[i]) continue;
    double work = (double)cnt[i] * threads * 8.0 * ITERS * ops_per_elem_iter;
    double r = work / (double)(hi[i] - lo[i]);
    rmin = r < rmin ? r : rmin; rmax = r > rmax ? r : rmax; rsum += r; ++nsm;
    if (hi[i] - lo[i] > span_max) span_max = hi[i] - lo[i];
  }
  printf("%-10s threads=%d ctas/SM=%d  SMs=%d  span=%lld cyc  ms=%.3f  => %.2f ops/clk/SM "
         "(SM min %.2f max %.2f; implied clock %.0f MHz)\n",
         name, threads, blocks_per_sm, nsm, span_max, ms, rsum / nsm, rmin, rmax,
         span_max / (ms * 1e3));
  cudaFree(out); cudaFree(cyc); delete[] h; delete[] lo; delete[] hi; delete[] cnt;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("%s SMs=%d cc=%d.%d\n", p.name, p.multiProcessorCount, p.major, p.minor);
  {
    double* d; cudaMalloc(&d, sizeof(double));
    const double rng[][2] = {{-1.0, 0.0}, {-30.0, 0.0}, {-126.0, -30.0}};
    for (auto& r : rng) {
      cudaMemset(d, 0, sizeof(double));
      k_ex2_acc<<<1184, 256>>>(r[0], r[1], 1LL << 26, d);
      double h; cudaMemcpy(&h, d, sizeof(double), cudaMemcpyDeviceToHost);
      printf("ex2.approx.ftz.f32 max rel err on [%g, %g]: %.3e (= 2^%.2f)\n", r[0], r[1], h, log2(h));
    }
    cudaFree(d);
  }
  for (int bps : {2, 4, 8}) {
    run("ex2+fadd", k_ex2, 1.0, 256, bps);       // counts ex2 per clk
    run("ex2", k_ex2_pure, 1.0, 256, bps);
    run("ffma", k_ffma, 2.0, 256, bps);          // FFMA lanes per clk
    run("ffma2", k_ffma2, 4.0, 256, bps);        // FP32 FMA lanes per clk (2 per FFMA2)
    run("ffma2_nr", k_ffma2_norreuse, 4.0, 256, bps);
    run("fwdmix", k_mix, 1.0, 256, bps);         // elements (pairs) per clk
  }
  return 0;
}
