// sf_launch.h -- internal launcher interface between the C-ABI (capi.cu) and
// the kernels (sf_kernels.cu, siddon_kernels.cu).  Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

#include "sf_common.cuh"

namespace ctp {

cudaError_t launch_transpose(const float* in, float* out, int R, int C, int batch,
                             cudaStream_t st);
// 3D pair.  xT: volume in [batch][ny*nx][nz] layout;
// sino: [batch][nv][nr][nc]
cudaError_t launch_forward(const GridParams& gp, const ViewCoef* vcoef, const ViewAx* vax, const float* xT,
                           float* sino, int batch, bool accumulate, cudaStream_t st);
// Back projection input (sino_prefix.cu): the sinogram [nviews][nr][nc] as
// [nviews][nc][nr] inclusive prefix sums over aligned kBackSeg-row segments
// of each column (raw, only transposed, with CTP_BACK_LEGACY); the in-place
// variant scans an already row-contiguous sinogram (FBP)
constexpr int kBackSeg = 128;
bool back_legacy();
cudaError_t launch_back_input(const float* sino, float* yT, int nr, int nc, int nviews, cudaStream_t st);
cudaError_t launch_back_input_inplace(float* yT, int nr, int nc, int nviews, cudaStream_t st);
// yT: sinogram from launch_back_input, [batch][nv][nc][nr]; vol: [batch][nz][ny][nx];
// only slices [z0, z1) of vol are written (z1 < 0: nz)
constexpr int kBackZBlock = 256;  // slices per back-kernel z-block (BK_ZC)
cudaError_t launch_back(const GridParams& gp, const ViewCoef* vcoef, const ViewAx* vax, const float* yT,
                        float* vol, int batch, bool accumulate, cudaStream_t st, int z0 = 0, int z1 = -1);
// round-1 3D back kernel (per-row overlaps), kept for A/B measurements
cudaError_t launch_back_legacy(const GridParams& gp, const ViewCoef* vcoef, const ViewAx* vax, const float* yT,
                               float* vol, int batch, bool accumulate, cudaStream_t st, int z0 = 0, int z1 = -1);
// round-1 3D forward kernel (per-row candidate overlaps), kept for A/B measurements
cudaError_t launch_forward_legacy(const GridParams& gp, const ViewCoef* vcoef, const ViewAx* vax, const float* xT,
                                  float* sino, int batch, bool accumulate, cudaStream_t st);
size_t forward_warp_smem_bytes();
// FBP input stage (ramp_kernels.cu): Ram-Lak filter of every detector row of
// in [nviews][nr][nc], times scale, written row-contiguous to out [nviews][nc][nr]
cudaError_t launch_ramp_rows_T(const float* in, float* out, int nr, int nc, int nviews, double pixel_width,
                               double scale, cudaStream_t st);
// fan beam (nz == nr == 1) with the batch on the lanes: inputs batch-innermost
// (xB [ny*nx][batch], yB [nv][nc][batch]), outputs in the natural layouts
// (sino [batch][nv][nc], vol [batch][ny*nx])
cudaError_t launch_forward_fan(const GridParams& gp, const ViewCoef* vcoef, const float* xB, float* sino,
                               int batch, cudaStream_t st);
cudaError_t launch_back_fan(const GridParams& gp, const ViewCoef* vcoef, const float* yB, float* vol,
                            int batch, cudaStream_t st);

// Siddon pair (siddon_kernels.cu): the float64 scalars of kernel_geom
// (_common.py:8-39) including the parallel-beam ray back-off `back`
struct SiddonParams {
  int kind, nv, nr, nc, nx, ny, nz;
  double pw, ph, cr, cc, sdd, back, x0, y0, z0, hx, hz;
};
// poses: device [nv][15] float64 (src, c0, u, vax, w); natural layouts
cudaError_t launch_siddon_forward(const SiddonParams& p, const double* poses, const float* vol, float* sino,
                                  int batch, bool accumulate, cudaStream_t st);
// ray_table: device scratch of siddon_ray_table_bytes(p) bytes, or nullptr to
// recompute the rays in the gather
size_t siddon_ray_table_bytes(const SiddonParams& p);
cudaError_t launch_siddon_back(const SiddonParams& p, const double* poses, const float* sino, float* vol,
                               int batch, bool accumulate, void* ray_table, cudaStream_t st);

}  // namespace ctp
