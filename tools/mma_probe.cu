// mma_probe.cu -- microbenchmark: legacy warp-level mma.sync m16n8k8 TF32 (SASS HMMA) on
// sm_100a: (1) throughput per SM, (2) input rounding (truncation vs round-to-nearest of the fp32
// operands' low 13 mantissa bits), (3) accumulation rounding over a long K chain, compared with
// an fp32 FMA chain and an fp64 reference. Development diagnostic for the forward's colour
// contraction.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_probe tools/mma_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4],
                                         const uint32_t (&b)[2]) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
        "{%8,%9}, {%0,%1,%2,%3};"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

template <int CH>
__global__ void k_tput(int iters, float* out, long long* cyc) {
    float d[CH][4] = {};
    uint32_t a[4], b[2];
    for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(1.0f + threadIdx.x * 1e-3f + i);
    b[0] = __float_as_uint(0.5f); b[1] = __float_as_uint(0.25f);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int c = 0; c < CH; ++c) mma_tf32(d[c], a, b);
    }
    long long t1 = clock64();
    float s = 0;
    for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// chain of K-steps: D += A_k B_k, A (16x8) and B (8x8) from global, one warp
__global__ void k_chain(const float* A, const float* B, int ksteps, float* D) {
    const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
    float d[4] = {0, 0, 0, 0};
    for (int k = 0; k < ksteps; ++k) {
        const float* Ak = A + (size_t)k * 128;   // row-major 16 x 8
        const float* Bk = B + (size_t)k * 64;    // row-major 8 (k) x 8 (n)
        uint32_t a[4] = {__float_as_uint(Ak[g * 8 + t]), __float_as_uint(Ak[(g + 8) * 8 + t]),
                         __float_as_uint(Ak[g * 8 + t + 4]), __float_as_uint(Ak[(g + 8) * 8 + t + 4])};
        uint32_t b[2] = {__float_as_uint(Bk[t * 8 + g]), __float_as_uint(Bk[(t + 4) * 8 + g])};
        mma_tf32(d, a, b);
    }
    D[g * 8 + 2 * t] = d[0];
    D[g * 8 + 2 * t + 1] = d[1];
    D[(g + 8) * 8 + 2 * t] = d[2];
    D[(g + 8) * 8 + 2 * t + 1] = d[3];
}

static float trunc13(float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xffffe000u; memcpy(&x, &u, 4); return x; }
static float rna13(float x) { uint32_t u; memcpy(&u, &x, 4); u += 0x1000u; u &= 0xffffe000u; memcpy(&x, &u, 4); return x; }

int main() {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    float* out; long long* cyc;
    cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 1 << 20);
    const int iters = 4096;
    for (int warps : {4, 8, 16}) {
        for (int blocks_per_sm : {1, 2, 4}) {
            int grid = sms * blocks_per_sm;
            k_tput<4><<<grid, 32 * warps>>>(iters, out, cyc);
            cudaDeviceSynchronize();
            std::vector<long long> c(grid);
            cudaMemcpy(c.data(), cyc, 8 * grid, cudaMemcpyDeviceToHost);
            double mx = 0; for (auto v : c) mx = fmax(mx, (double)v);
            double macs = (double)iters * 4 * 16 * 8 * 8 * warps * blocks_per_sm;
            printf("tput: warps/CTA %2d CTAs/SM %d: %.1f MAC/clk/SM (%.2f cyc per mma per SMSP)\n",
                   warps, blocks_per_sm, macs / mx,
                   mx / ((double)iters * 4 * warps * blocks_per_sm / 4));
        }
    }
    // precision: K chain of random values in [0,1) (A) and [0,0.5) (B)
    for (int mode = 0; mode < 3; ++mode) {
        const int ks = 512;
        std::vector<float> A(ks * 128), B(ks * 64);
        srand(1 + mode);
        for (auto& x : A) { x = (float)rand() / RAND_MAX; if (mode == 0) x = trunc13(x); }
        for (auto& x : B) { x = 0.5f * (float)rand() / RAND_MAX; if (mode == 0) x = trunc13(x); }
        float *dA, *dB, *dD;
        cudaMalloc(&dA, 4 * A.size()); cudaMalloc(&dB, 4 * B.size()); cudaMalloc(&dD, 4 * 128);
        cudaMemcpy(dA, A.data(), 4 * A.size(), cudaMemcpyHostToDevice);
        cudaMemcpy(dB, B.data(), 4 * B.size(), cudaMemcpyHostToDevice);
        k_chain<<<1, 32>>>(dA, dB, ks, dD);
        std::vector<float> D(128);
        cudaMemcpy(D.data(), dD, 4 * 128, cudaMemcpyDeviceToHost);
        double e_ref = 0, e_trunc = 0, e_rna = 0, e_f32 = 0, mag = 0;
        for (int m = 0; m < 16; ++m)
            for (int n = 0; n < 8; ++n) {
                double ex = 0, et = 0, er = 0;
                float f32 = 0;
                for (int k = 0; k < ks; ++k)
                    for (int j = 0; j < 8; ++j) {
                        float a = A[k * 128 + m * 8 + j], b = B[k * 64 + j * 8 + n];
                        ex += (double)a * b;
                        et += (double)trunc13(a) * trunc13(b);
                        er += (double)rna13(a) * rna13(b);
                        f32 = fmaf(a, b, f32);
                    }
                mag = fmax(mag, fabs(ex));
                e_ref = fmax(e_ref, fabs(D[m * 8 + n] - ex) / fabs(ex));
                e_trunc = fmax(e_trunc, fabs(D[m * 8 + n] - et) / fabs(et));
                e_rna = fmax(e_rna, fabs(D[m * 8 + n] - er) / fabs(er));
                e_f32 = fmax(e_f32, fabs(f32 - ex) / fabs(ex));
            }
        printf("precision mode %d (%s inputs, K=%d): max rel err vs exact %.3e | vs exact-of-truncated "
               "inputs %.3e | vs exact-of-RNA inputs %.3e | fp32 FMA chain vs exact %.3e (|D|~%.1f)\n",
               mode, mode == 0 ? "tf32-exact" : "full fp32", ks * 8, e_ref, e_trunc, e_rna, e_f32,
               mag);
    }
    return 0;
}
