// sino_prefix.cu -- input stage of the 3D SF back projection: the sinogram
// in the row-contiguous layout [nv][nc][nr] the back kernel reads, as
// INCLUSIVE PREFIX SUMS over the rows of each aligned 128-row segment
//
//   I(r) = sum_{r' = 128 floor(r / 128)}^{r} y(r'),
//
// so the back kernel's per-(voxel column, view) table of running row sums
// (sf_back3d.cu) is a weighted sum of I plus one carry per segment, with no
// warp scans of its own.  The segments bound the magnitudes summed in fp32
// (128 rows), and a raw value is I(r) - I(r - 1) inside a segment.
//
// transpose_segscan_kernel fuses the layout change [nv][nr][nc] -> [nv][nc][nr]
// (it replaces the plain transpose: same traffic, one read and one write of
// the sinogram); segscan_rows_kernel scans an already row-contiguous sinogram
// in place (the FBP path, after ramp_rows_T_kernel).  With CTP_BACK_LEGACY
// set (A/B against round 1's per-row kernel) the input stays raw.
#include <cuda_runtime.h>

#include <cstdlib>

#include "sf_launch.h"

namespace ctp {

namespace {
constexpr int SEG = kBackSeg;   // rows per segment
constexpr int TS_WARPS = 8;     // warps per CTA, one (view, 32-column strip, segment) each
}  // namespace

bool back_legacy() {
  static const bool legacy = getenv("CTP_BACK_LEGACY") != nullptr;
  return legacy;
}

// One warp: 32 columns (lane = column) x one segment, in 32-row sub-blocks:
// coalesced row reads, a running sum per lane, and the transposed write-out
// through a 32 x 33 shared tile (conflict-free both ways).
__global__ void __launch_bounds__(TS_WARPS * 32) transpose_segscan_kernel(const float* __restrict__ in,
                                                                          float* __restrict__ out, int nr, int nc,
                                                                          long long ntasks) {
  __shared__ float tile[TS_WARPS][32][33];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long task = (long long)blockIdx.x * TS_WARPS + warp;
  if (task >= ntasks) return;  // warp-uniform; no CTA barriers
  const int nstrip = (nc + 31) >> 5, nseg = (nr + SEG - 1) / SEG;
  const int strip = (int)(task % nstrip);
  const long long t2 = task / nstrip;
  const int seg = (int)(t2 % nseg);
  const long long v = t2 / nseg;
  const int c0 = strip * 32;
  const int c = c0 + lane;
  const float* src = in + (size_t)v * nr * nc + c;
  float* dst = out + (size_t)v * nc * nr;
  float(&T)[32][33] = tile[warp];
  float run = 0.0f;
#pragma unroll 1
  for (int sb = 0; sb < SEG / 32; ++sb) {
    const int r0 = seg * SEG + sb * 32;
    if (r0 >= nr) break;
    float vals[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) vals[i] = (c < nc && r0 + i < nr) ? __ldg(src + (size_t)(r0 + i) * nc) : 0.0f;
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      run += vals[i];
      T[lane][i] = run;
    }
    __syncwarp();
    const int nrow = min(32, nr - r0);
    const int ncol = min(32, nc - c0);
    for (int cc = 0; cc < ncol; ++cc)
      if (lane < nrow) dst[(size_t)(c0 + cc) * nr + r0 + lane] = T[cc][lane];
    __syncwarp();
  }
}

// One warp: one (view, column, segment), lane t owns rows 4 t .. 4 t + 3 of
// the segment: local prefix, warp scan of the lane totals, in place.
__global__ void __launch_bounds__(256) segscan_rows_kernel(float* __restrict__ y, int nr, long long ntasks) {
  const int lane = threadIdx.x & 31;
  const long long task = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (task >= ntasks) return;
  const int nseg = (nr + SEG - 1) / SEG;
  const long long col = task / nseg;  // (view, column)
  const int seg = (int)(task % nseg);
  float* p = y + (size_t)col * nr + seg * SEG + 4 * lane;
  const int r = seg * SEG + 4 * lane;
  float q[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) q[i] = r + i < nr ? p[i] : 0.0f;
  q[1] += q[0];
  q[2] += q[1];
  q[3] += q[2];
  float inc = q[3];
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const float n = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += n;
  }
  const float ex = inc - q[3];
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (r + i < nr) p[i] = ex + q[i];
}

cudaError_t launch_back_input(const float* sino, float* yT, int nr, int nc, int nviews, cudaStream_t st) {
  if (back_legacy()) return launch_transpose(sino, yT, nr, nc, nviews, st);
  if (nr < 1 || nc < 1 || nviews < 1) return cudaErrorInvalidValue;
  const long long ntasks = (long long)nviews * ((nr + SEG - 1) / SEG) * ((nc + 31) / 32);
  const long long nblocks = (ntasks + TS_WARPS - 1) / TS_WARPS;
  if (nblocks > 0x7fffffffLL) return cudaErrorInvalidValue;
  transpose_segscan_kernel<<<(unsigned)nblocks, TS_WARPS * 32, 0, st>>>(sino, yT, nr, nc, ntasks);
  return cudaGetLastError();
}

cudaError_t launch_back_input_inplace(float* yT, int nr, int nc, int nviews, cudaStream_t st) {
  if (back_legacy()) return cudaSuccess;
  if (nr < 1 || nc < 1 || nviews < 1) return cudaErrorInvalidValue;
  const long long ntasks = (long long)nviews * nc * ((nr + SEG - 1) / SEG);
  const long long nblocks = (ntasks + 7) / 8;
  if (nblocks > 0x7fffffffLL) return cudaErrorInvalidValue;
  segscan_rows_kernel<<<(unsigned)nblocks, 256, 0, st>>>(yT, nr, ntasks);
  return cudaGetLastError();
}

}  // namespace ctp
