// Device-side helpers: CSR-order stencil rows and deterministic block reductions.
#pragma once

#include <cuda_runtime.h>

namespace pint {

// Row sum of a 9-point stencil at interior point (x, y) of plane v (m x m),
// in CSR column order SW,S,SE,W,C,E,NW,N,NE; neighbours outside the grid
// contribute a*0 (exact).  Matches scipy csr_matvec (linalg.py:96-97):
// sum = 0; sum += a_k * x_k in column order.  Requires -fmad=false.
__device__ __forceinline__ double stencil9_global(const double* __restrict__ c,
                                                  const double* __restrict__ v, int m, int x,
                                                  int y) {
    const int i = y * m + x;
    const bool w = x > 0, e = x < m - 1, s = y > 0, nn = y < m - 1;
    const double t0 = (s && w) ? __ldg(v + i - m - 1) : 0.0;
    const double t1 = s ? __ldg(v + i - m) : 0.0;
    const double t2 = (s && e) ? __ldg(v + i - m + 1) : 0.0;
    const double t3 = w ? __ldg(v + i - 1) : 0.0;
    const double t4 = __ldg(v + i);
    const double t5 = e ? __ldg(v + i + 1) : 0.0;
    const double t6 = (nn && w) ? __ldg(v + i + m - 1) : 0.0;
    const double t7 = nn ? __ldg(v + i + m) : 0.0;
    const double t8 = (nn && e) ? __ldg(v + i + m + 1) : 0.0;
    double r = c[0] * t0;
    r = r + c[1] * t1;
    r = r + c[2] * t2;
    r = r + c[3] * t3;
    r = r + c[4] * t4;
    r = r + c[5] * t5;
    r = r + c[6] * t6;
    r = r + c[7] * t7;
    r = r + c[8] * t8;
    return r;
}

// Same row sum over a shared-memory tile with row pitch P; (ly, lx) is the
// centre's local position, zero padding outside the grid already in place.
template <int P>
__device__ __forceinline__ double stencil9_smem(const double* c, const double* t, int ly,
                                                int lx) {
    const double* r0 = t + (ly - 1) * P + lx;
    const double* r1 = t + ly * P + lx;
    const double* r2 = t + (ly + 1) * P + lx;
    double r = c[0] * r0[-1];
    r = r + c[1] * r0[0];
    r = r + c[2] * r0[1];
    r = r + c[3] * r1[-1];
    r = r + c[4] * r1[0];
    r = r + c[5] * r1[1];
    r = r + c[6] * r2[-1];
    r = r + c[7] * r2[0];
    r = r + c[8] * r2[1];
    return r;
}

// Deterministic block sum (fixed shuffle tree); result valid in thread 0.
template <int NT>
__device__ __forceinline__ double block_sum(double v) {
    __shared__ double warp_part[NT / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int tid = threadIdx.x + threadIdx.y * blockDim.x;
    if ((tid & 31) == 0) warp_part[tid >> 5] = v;
    __syncthreads();
    double s = 0.0;
    if (tid == 0) {
#pragma unroll
        for (int w = 0; w < NT / 32; ++w) s += warp_part[w];
    }
    return s;
}

}  // namespace pint
