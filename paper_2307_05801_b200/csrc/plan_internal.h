// plan_internal.h -- the ctp_plan object and error helpers shared by the
// C-ABI translation units (capi.cu, dist.cu).  Not part of the public ABI.
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "../../include/ctproj_b200.h"
#include "sf_common.cuh"

struct ctp_plan {
  ctp_geom geom;               // scalars (poses pointer cleared)
  std::vector<double> poses;   // host copy, nv*15
  int device;
  ctp::ViewCoef* d_coef;            // device, nv entries
  ctp::ViewAx* d_ax;                // device, nv entries (f64 axial map of the 3D kernels)
  double* d_pose;              // device, nv*15 float64 (Siddon pair)
  bool sf_ok;                  // SF supports this geometry (SF-modular: upright panels only)
  std::string sf_reason;
  ctp::GridParams gp;
  size_t vol_elems, sino_elems;
  cudaEvent_t ev[2][2];        // [direction][start/stop], created lazily
  bool ev_recorded[2];
};


namespace ctp_internal {

extern thread_local std::string g_last_error;
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);

struct DeviceGuard {
  int prev = -1;
  bool switched = false;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    err = cudaGetDevice(&prev);
    if (err == cudaSuccess && dev >= 0 && dev != prev) {
      err = cudaSetDevice(dev);
      switched = (err == cudaSuccess);
    }
  }
  ~DeviceGuard() {
    if (switched) cudaSetDevice(prev);
  }
};

}  // namespace ctp_internal
