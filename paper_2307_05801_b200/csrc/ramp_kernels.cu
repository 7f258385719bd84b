// ramp_kernels.cu -- FBP input stage: Ram-Lak ramp
// filter of every detector row, fused with the [nv][nr][nc] -> [nv][nc][nr]
// layout change the SF back kernel reads (it replaces the back projection's
// transpose pass), so FBP = this kernel + the back projection kernel.
//
// Reference: ramp_filter_rows / _ramp_kernel, pkg/src/ctproj/recon.py:39-61.
// The reference convolves each row with the discrete Ram-Lak kernel
//   h[0] = 1 / (4 d^2),  h[m] = -1 / (pi m d)^2 (m odd),  h[m] = 0 (m even, != 0)
// through a float64 FFT zero-padded to n >= 2 nc; with that padding the
// circular convolution equals the LINEAR convolution out[c] = sum_p h[c - p] in[p]
// over |c - p| < nc, which this kernel evaluates directly in fp32 (a few
// hundred decaying terms per output, ~1e-7 relative to the f64 FFT).
//
// Tiling: a CTA owns RB consecutive rows of one view (all nc columns) in shared
// memory (row stride nc + 1: conflict-free per-row reads); a thread owns one
// row and 8 consecutive output columns, and walks the inputs in 8 x 8 blocks
// whose kernel offsets m = c - p have a static parity (c and p start at
// multiples of 8), so the zero taps of even m are skipped at compile time
// (m = 0 only on the diagonal block).  Output writes are coalesced along rows.
#include <cuda_runtime.h>

#include <cmath>

#include "sf_launch.h"

namespace ctp {

template <int RB>
__global__ void __launch_bounds__(256) ramp_rows_T_kernel(const float* __restrict__ in, float* __restrict__ out,
                                                          int nr, int nc, float h0, float hs, float scale) {
  extern __shared__ float ramp_smem[];
  const int ncp = nc + 1;
  float* tile = ramp_smem;              // [RB][nc + 1]
  float* hodd = ramp_smem + RB * ncp;   // hodd[m + nc] = h[m] for odd m, m in (-nc, nc)
  const int v = blockIdx.y;             // view (x batch)
  const int r0 = blockIdx.x * RB;
  const float* src = in + (size_t)v * nr * nc;
  for (int i = threadIdx.x; i < RB * nc; i += blockDim.x) {
    const int rr = i / nc, c = i - rr * nc;
    tile[rr * ncp + c] = (r0 + rr < nr) ? __ldg(src + (size_t)(r0 + rr) * nc + c) : 0.0f;
  }
  for (int m = threadIdx.x; m < 2 * nc; m += blockDim.x) {
    const int k = m - nc;
    const float kf = (float)k;
    hodd[m] = (k & 1) ? hs / (kf * kf) : 0.0f;  // hs = -1 / (pi d)^2
  }
  __syncthreads();
  const int r = threadIdx.x % RB;
  const int groups = blockDim.x / RB;
  const float* row = tile + r * ncp;
  float* dst = out + (size_t)v * nc * nr + r0 + r;
  const bool live = r0 + r < nr;
  const int nch = (nc + 7) / 8;
  for (int ch = threadIdx.x / RB; ch < nch; ch += groups) {
    const int c0 = 8 * ch;
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.0f;
    for (int p0 = 0; p0 < nc; p0 += 8) {
      float x[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = (p0 + i < nc) ? row[p0 + i] : 0.0f;
      // taps m = c0 - p0 + (j - i), j - i odd: hodd[c0 - p0 + d + nc], d = -7, -5, ..., 7
      const float* hb = hodd + (c0 - p0 + nc);
      float h[15];
#pragma unroll
      for (int d = -7; d <= 7; d += 2) h[d + 7] = (c0 - p0 + d > -nc && c0 - p0 + d < nc) ? hb[d] : 0.0f;
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int i = 0; i < 8; ++i)
          if ((j - i) & 1) acc[j] = fmaf(h[j - i + 7], x[i], acc[j]);
      if (p0 == c0) {  // diagonal block: the m = 0 tap
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] = fmaf(h0, x[j], acc[j]);
      }
    }
    if (live) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (c0 + j < nc) dst[(size_t)(c0 + j) * nr] = acc[j] * scale;
    }
  }
}

cudaError_t launch_ramp_rows_T(const float* in, float* out, int nr, int nc, int nviews, double pixel_width,
                               double scale, cudaStream_t st) {
  if (nr < 1 || nc < 1 || nviews < 1 || !(pixel_width > 0.0)) return cudaErrorInvalidValue;
  const float h0 = (float)(1.0 / (4.0 * pixel_width * pixel_width));
  const float hs = (float)(-1.0 / (M_PI * M_PI * pixel_width * pixel_width));
  int rb = 32;
  while (rb > 8 && (size_t)(rb * (nc + 1) + 2 * nc) * sizeof(float) > 200 * 1024) rb /= 2;
  const size_t smem = (size_t)(rb * (nc + 1) + 2 * nc) * sizeof(float);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  for (int v0 = 0; v0 < nviews; v0 += 65535) {
    const int nv = nviews - v0 < 65535 ? nviews - v0 : 65535;
    const dim3 grid((nr + rb - 1) / rb, nv);
    const float* i0 = in + (size_t)v0 * nr * nc;
    float* o0 = out + (size_t)v0 * nr * nc;
    cudaError_t e = cudaSuccess;
    switch (rb) {
      case 32:
        e = cudaFuncSetAttribute(ramp_rows_T_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess)
          ramp_rows_T_kernel<32><<<grid, 256, smem, st>>>(i0, o0, nr, nc, h0, hs, (float)scale);
        break;
      case 16:
        e = cudaFuncSetAttribute(ramp_rows_T_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess)
          ramp_rows_T_kernel<16><<<grid, 256, smem, st>>>(i0, o0, nr, nc, h0, hs, (float)scale);
        break;
      default:
        e = cudaFuncSetAttribute(ramp_rows_T_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess)
          ramp_rows_T_kernel<8><<<grid, 256, smem, st>>>(i0, o0, nr, nc, h0, hs, (float)scale);
        break;
    }
    if (e != cudaSuccess) return e;
  }
  return cudaGetLastError();
}

}  // namespace ctp
