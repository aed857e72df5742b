// train.cu -- NEXT-1: the training-step adjacency of the rasterizer, fused.
//
// Gaussian Primary Head activations: alpha = sigmoid(raw_alpha),
// c = sigmoid(raw_c), sigma = sigmoid(raw_sigma), rho = rho_scale * tanh(raw_rho) (the paper's
// tanh is rho_scale = 1; SPEC's rho_eps reading is rho_scale = 1 - 1e-4), mu = p + o with the
// reference position p supplied by the caller. The L1 loss against the HR ground truth
// is fused into the forward epilogue (sum |I - I_gt|) and its gradient
// sign(I - I_gt) / numel into the backward's dL/dI staging, so no gradient image is materialised.
#include "gsr_internal.cuh"

namespace gsr {

namespace {

__device__ __forceinline__ float sigmoidf_acc(float x) { return 1.0f / (1.0f + expf(-x)); }

__global__ void k_activate(const float* __restrict__ raw_alpha, const float* __restrict__ offset,
                           const float* __restrict__ ref, const float* __restrict__ raw_sigma,
                           const float* __restrict__ raw_rho, const float* __restrict__ raw_color,
                           long long n, float rho_scale, float* __restrict__ alpha,
                           float* __restrict__ mu, float* __restrict__ sigma,
                           float* __restrict__ rho, float* __restrict__ color) {
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    alpha[i] = sigmoidf_acc(raw_alpha[i]);
    mu[2 * i] = ref[2 * i] + offset[2 * i];
    mu[2 * i + 1] = ref[2 * i + 1] + offset[2 * i + 1];
    sigma[2 * i] = sigmoidf_acc(raw_sigma[2 * i]);
    sigma[2 * i + 1] = sigmoidf_acc(raw_sigma[2 * i + 1]);
    rho[i] = rho_scale * tanhf(raw_rho[i]);
    color[3 * i] = sigmoidf_acc(raw_color[3 * i]);
    color[3 * i + 1] = sigmoidf_acc(raw_color[3 * i + 1]);
    color[3 * i + 2] = sigmoidf_acc(raw_color[3 * i + 2]);
}

__global__ void k_scale(double* v, double s) { *v *= s; }

}  // namespace

cudaError_t launch_activate(const float* raw_alpha, const float* offset, const float* ref,
                            const float* raw_sigma, const float* raw_rho, const float* raw_color,
                            long long n, float rho_scale, float* alpha, float* mu, float* sigma,
                            float* rho, float* color, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    count_launches(1);
    k_activate<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(raw_alpha, offset, ref, raw_sigma,
                                                            raw_rho, raw_color, n, rho_scale,
                                                            alpha, mu, sigma, rho, color);
    return cudaGetLastError();
}

cudaError_t launch_scale_loss(double* loss, double scale, cudaStream_t st) {
    count_launches(1);
    k_scale<<<1, 1, 0, st>>>(loss, scale);
    return cudaGetLastError();
}

}  // namespace gsr
