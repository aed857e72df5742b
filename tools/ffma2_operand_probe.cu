// FFMA2 operand-form probe (development, compile-only): which operands ptxas feeds from uniform
// registers. Build and inspect the SASS:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -cubin -o /tmp/p.cubin tools/ffma2_operand_probe.cu
//   cuobjdump -sass /tmp/p.cubin | grep -E "FFMA2|REDUX|MOV"
// k_param: a kernel parameter is read straight from a uniform register
//          (FFMA2 R22, R10.F32x2.HI_LO, UR6.F32, R22.F32x2.HI_LO: two vector pairs -> rt 2).
// k_redux: a per-iteration warp-uniform value (REDUX.OR into a UR) is moved back to a vector
//          register (MOV R21, UR5) before the FFMA2 -> pair + scalar + pair -> rt 3.
#include <cuda_runtime.h>

__global__ void k_param(const float2* __restrict__ e, float2* out, int n, float p, float q) {
    float2 acc = make_float2(0.f, 0.f);
    for (int i = 0; i < n; ++i) {
        float2 ev = e[i * 32 + threadIdx.x];
        acc = __ffma2_rn(make_float2(p, p), ev, acc);
        acc = __ffma2_rn(make_float2(q, q), ev, acc);
    }
    out[threadIdx.x] = acc;
}

__device__ __forceinline__ float unif(float x) {
    return __int_as_float(__reduce_or_sync(0xffffffffu, __float_as_int(x)));
}

__global__ void k_redux(const float* __restrict__ g, const float2* __restrict__ e, float2* out,
                        int n) {
    float2 acc = make_float2(0.f, 0.f), acc2 = acc, acc3 = acc;
    for (int i = 0; i < n; ++i) {
        float gr = unif(g[3 * i]), gg = unif(g[3 * i + 1]), gb = unif(g[3 * i + 2]);
        float2 ev = e[i * 32 + threadIdx.x];
        acc = __ffma2_rn(ev, make_float2(gr, gr), acc);
        acc2 = __ffma2_rn(ev, make_float2(gg, gg), acc2);
        acc3 = __ffma2_rn(ev, make_float2(gb, gb), acc3);
    }
    out[threadIdx.x] = acc;
    out[threadIdx.x + 32] = acc2;
    out[threadIdx.x + 64] = acc3;
}
