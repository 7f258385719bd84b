// capi.cu -- extern "C" boundary of libctproj_b200.so (include/ctproj_b200.h).
//
// Host side of the drop-in: validates the flattened geometry (what
// kernel_geom()/pose_table() produce, _common.py:8-39, geometry.py:227-263),
// digests it in float64 into per-view footprint coefficients (ViewCoef,
// sf_common.cuh) that stay resident on the device, and launches the SF
// kernels stream-ordered.  No host synchronisation on the hot path.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/ctproj_b200.h"
#include "sf_common.cuh"
#include "sf_launch.h"

using ctp::GridParams;
using ctp::ViewAx;
using ctp::ViewCoef;

#include "plan_internal.h"

namespace ctp_internal {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  g_last_error = std::string(where) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? CTP_ERR_OUT_OF_MEMORY : CTP_ERR_CUDA;
}

}  // namespace ctp_internal

using ctp_internal::DeviceGuard;
using ctp_internal::cuda_fail;
using ctp_internal::fail;
using ctp_internal::g_last_error;

namespace {

int validate(const ctp_geom* g) {
  if (!g) return fail(CTP_ERR_INVALID_ARGUMENT, "geometry pointer is null");
  if (g->kind < CTP_PARALLEL || g->kind > CTP_MODULAR)
    return fail(CTP_ERR_INVALID_ARGUMENT, "unknown geometry kind");
  if (g->num_views < 1 || g->num_rows < 1 || g->num_cols < 1)
    return fail(CTP_ERR_INVALID_ARGUMENT, "detector/view counts must be >= 1");
  if (g->num_x < 1 || g->num_y < 1 || g->num_z < 1)
    return fail(CTP_ERR_INVALID_ARGUMENT, "voxel counts must be >= 1");
  if (!(g->pixel_width > 0 && g->pixel_height > 0))
    return fail(CTP_ERR_INVALID_ARGUMENT, "pixel sizes must be > 0");
  if (!(g->voxel_width > 0 && g->voxel_height > 0))
    return fail(CTP_ERR_INVALID_ARGUMENT, "voxel sizes must be > 0");
  if ((g->kind == CTP_CONE_FLAT || g->kind == CTP_CONE_CURVED) && !(g->sdd > 0))
    return fail(CTP_ERR_INVALID_ARGUMENT, "cone geometry requires sdd > 0");
  if (!g->poses) return fail(CTP_ERR_INVALID_ARGUMENT, "pose table pointer is null");
  if (g->num_x > 65535 || g->num_y > 65535)
    return fail(CTP_ERR_INVALID_ARGUMENT, "grid too large (nx, ny <= 65535)");
  const long long nvox = (long long)g->num_x * g->num_y * g->num_z;
  const long long nsino = (long long)g->num_views * g->num_rows * g->num_cols;
  if (nvox >= (1LL << 40) || nsino >= (1LL << 40))
    return fail(CTP_ERR_INVALID_ARGUMENT, "array too large");
  for (long long k = 0; k < 15LL * g->num_views; ++k)
    if (!std::isfinite(g->poses[k])) return fail(CTP_ERR_INVALID_ARGUMENT, "non-finite pose entry");
  return CTP_OK;
}

// SF-modular (an extension: the reference raises UnsupportedGeometryError for
// SF + modular, sf.py:23-27) is exact only for UPRIGHT panels: detector
// columns horizontal (colDir.z = 0) and rows vertical (rowDir = +z), in any
// position and yaw, with the source anywhere.  Then the detector normal is
// horizontal, a voxel column's transverse footprint does not move with z and
// its axial map is affine in z, exactly as for cone-flat.  A tilted panel
// would need a z-dependent transverse footprint (non-separable), so it is
// rejected here instead of being approximated; the Siddon pair supports every
// modular pose.
constexpr double kUprightTol = 1e-6;
bool sf_supports(const ctp_geom* g) {
  if (g->kind != CTP_MODULAR) return true;
  for (int v = 0; v < g->num_views; ++v) {
    const double* P = g->poses + 15 * v;
    const double uz = P[8], vx = P[9], vy = P[10], vz = P[11];
    if (!(std::fabs(uz) <= kUprightTol && std::fabs(vx) <= kUprightTol && std::fabs(vy) <= kUprightTol &&
          vz > 0.0))
      return false;
  }
  return true;
}

// float64 digestion of one view's pose into affine footprint coefficients
// over centred grid-index coordinates (see sf_common.cuh for the frame).
void build_view_coefs(const ctp_geom& g, const double* P, std::vector<ViewCoef>& out,
                      std::vector<ViewAx>& axo) {
  const double hx = g.voxel_width, hz = g.voxel_height;
  const double pw = g.pixel_width, ph = g.pixel_height, cr = g.center_row, cc = g.center_col;
  const double xm = g.x0 + 0.5 * g.num_x * hx, ym = g.y0 + 0.5 * g.num_y * hx;
  const double half_x = 0.5 * g.num_x, half_y = 0.5 * g.num_y;
  out.assign(g.num_views, ViewCoef{});
  axo.assign(g.num_views, ViewAx{});
  for (int v = 0; v < g.num_views; ++v) {
    const double* s = P + 15 * v;
    const double* c0 = s + 3;
    const double* u = s + 6;
    const double* vax = s + 9;
    const double* w = s + 12;
    ViewCoef& c = out[v];
    ViewAx& ax = axo[v];
    c.ux = (float)u[0];
    c.uy = (float)u[1];
    c.wx = (float)w[0];
    c.wy = (float)w[1];
    c.xs = (float)((s[0] - xm) / hx);
    c.ys = (float)((s[1] - ym) / hx);
    c.xc0 = (float)((c0[0] - xm) / hx);
    c.yc0 = (float)((c0[1] - ym) / hx);
    // _sf_subdivide (_kernels.py:550): the tie at 45 deg must be broken in f64
    c.split_x = (std::fabs(u[0]) * hx >= std::fabs(u[1]) * hx) ? 1 : 0;
    if (g.kind == CTP_PARALLEL) {
      // s = (p - c0).u at z = 0 (_kernels.py:457-460), T = tcen/ph + cr (:621-625)
      c.na = (float)(((xm - c0[0]) * u[0] + (ym - c0[1]) * u[1] - c0[2] * u[2]) / pw + cc);
      c.nb = (float)(hx * u[0] / pw);
      c.nc = (float)(hx * u[1] / pw);
      c.ta = (float)(((xm - c0[0]) * vax[0] + (ym - c0[1]) * vax[1] +
                      (g.z0 + 0.5 * hz - c0[2]) * vax[2]) / ph + cr);
      c.tb = (float)(hx * vax[0] / ph);
      c.tc = (float)(hx * vax[1] / ph);
      c.tz = (float)(hz * vax[2] / ph);
      c.cull = 1;
      ax.k0 = 1.0;  // mag = 1
      ax.lam = 1.0;
      ax.a0 = ((xm - c0[0]) * vax[0] + (ym - c0[1]) * vax[1] + (g.z0 + 0.5 * hz - c0[2]) * vax[2]) / ph + cr;
      ax.a2 = hx * vax[0] / ph;
      ax.a3 = hx * vax[1] / ph;
      ax.bz = hz * vax[2] / ph;
      continue;
    }
    if (g.kind == CTP_MODULAR) {
      // flat panel in an arbitrary pose (extension): the
      // transverse trapezoid is taken at the grid's centre height zr with the
      // full 3-D ray/plane intersection, the axial map from the column centre
      // line (affine in z for a detector whose normal is horizontal)
      const double nxv = u[1] * vax[2] - u[2] * vax[1];
      const double nyv = u[2] * vax[0] - u[0] * vax[2];
      const double nzv = u[0] * vax[1] - u[1] * vax[0];
      const double lamnum = (c0[0] - s[0]) * nxv + (c0[1] - s[1]) * nyv + (c0[2] - s[2]) * nzv;
      const double zr = g.z0 + 0.5 * g.num_z * hz;
      c.dxa = (float)(xm - s[0]);
      c.dya = (float)(ym - s[1]);
      c.zc0 = (float)(g.z0 + 0.5 * hz - s[2]);
      c.na = (float)((xm - s[0]) * u[0] + (ym - s[1]) * u[1] + (zr - s[2]) * u[2]);
      c.nb = (float)(hx * u[0]);
      c.nc = (float)(hx * u[1]);
      c.da = (float)((xm - s[0]) * nxv + (ym - s[1]) * nyv + (zr - s[2]) * nzv);
      c.db = (float)(hx * nxv);
      c.dc = (float)(hx * nyv);
      c.dm = c.da;
      c.s0 = (float)(((s[0] - c0[0]) * u[0] + (s[1] - c0[1]) * u[1] + (s[2] - c0[2]) * u[2]) / pw + cc);
      c.g = (float)(lamnum / pw);
      c.lamnum = (float)lamnum;
      c.ta = (float)(((s[0] - c0[0]) * vax[0] + (s[1] - c0[1]) * vax[1] + (s[2] - c0[2]) * vax[2]) / ph + cr);
      c.tb = (float)(hx * vax[0] / ph);
      c.tc = (float)(hx * vax[1] / ph);
      c.tz = (float)vax[2];
      c.tva = (float)(((xm - s[0]) * vax[0] + (ym - s[1]) * vax[1]) / ph);
      const bool inside = std::fabs((s[0] - xm) / hx) < half_x + 2.0 &&
                          std::fabs((s[1] - ym) / hx) < half_y + 2.0;
      c.cull = inside ? 0 : 1;
      ax.k0 = (xm - s[0]) * nxv + (ym - s[1]) * nyv + (zr - s[2]) * nzv;
      ax.k1 = hx * nxv;
      ax.k2 = hx * nyv;
      ax.lam = lamnum;
      ax.a0 = ((s[0] - c0[0]) * vax[0] + (s[1] - c0[1]) * vax[1] + (s[2] - c0[2]) * vax[2]) / ph + cr;
      ax.a1 = vax[2] * (g.z0 + 0.5 * hz - s[2]) / ph + ((xm - s[0]) * vax[0] + (ym - s[1]) * vax[1]) / ph;
      ax.a2 = hx * vax[0] / ph;
      ax.a3 = hx * vax[1] / ph;
      ax.bz = vax[2] * hz / ph;
      continue;
    }
    // cone: plane normal and lamnum (_kernels.py:562-569)
    const double nxv = u[1] * vax[2] - u[2] * vax[1];
    const double nyv = u[2] * vax[0] - u[0] * vax[2];
    const double nzv = u[0] * vax[1] - u[1] * vax[0];
    const double lamnum = (c0[0] - s[0]) * nxv + (c0[1] - s[1]) * nyv + (c0[2] - s[2]) * nzv;
    c.dxa = (float)(xm - s[0]);
    c.dya = (float)(ym - s[1]);
    c.zc0 = (float)(g.z0 + 0.5 * hz - s[2]);
    if (g.kind == CTP_CONE_FLAT) {
      c.na = (float)((xm - s[0]) * u[0] + (ym - s[1]) * u[1] - s[2] * u[2]);
      c.nb = (float)(hx * u[0]);
      c.nc = (float)(hx * u[1]);
      c.da = (float)((xm - s[0]) * nxv + (ym - s[1]) * nyv - s[2] * nzv);
      c.db = (float)(hx * nxv);
      c.dc = (float)(hx * nyv);
      c.dm = (float)((xm - s[0]) * nxv + (ym - s[1]) * nyv);
      c.s0 = (float)(((s[0] - c0[0]) * u[0] + (s[1] - c0[1]) * u[1] + (s[2] - c0[2]) * u[2]) / pw + cc);
      c.g = (float)(lamnum / pw);
      c.lamnum = (float)lamnum;
      ax.k0 = (xm - s[0]) * nxv + (ym - s[1]) * nyv;
      ax.k1 = hx * nxv;
      ax.k2 = hx * nyv;
      ax.lam = lamnum;
    } else {  // curved: s = sdd * atan2(e.u, e.w) (_kernels.py:478-497)
      c.na = (float)((xm - s[0]) * u[0] + (ym - s[1]) * u[1]);
      c.nb = (float)(hx * u[0]);
      c.nc = (float)(hx * u[1]);
      c.da = (float)((xm - s[0]) * w[0] + (ym - s[1]) * w[1]);
      c.db = (float)(hx * w[0]);
      c.dc = (float)(hx * w[1]);
      c.s0 = (float)cc;
      c.g = (float)(g.sdd / pw);
      c.lamnum = (float)g.sdd;
      ax.k0 = xm - s[0];
      ax.k1 = ym - s[1];
      ax.k2 = hx;
      ax.lam = g.sdd;
    }
    // cone axial map: tcen = mag (cz - src_z) (_kernels.py:626-628) in row units
    ax.a0 = cr;
    ax.a1 = (g.z0 + 0.5 * hz - s[2]) / ph;
    ax.bz = hz / ph;
    // wedge culling assumes the source lies outside the grid footprint
    const bool inside = std::fabs((s[0] - xm) / hx) < half_x + 2.0 &&
                        std::fabs((s[1] - ym) / hx) < half_y + 2.0;
    c.cull = inside ? 0 : 1;
  }
}

GridParams make_grid_params(const ctp_geom& g) {
  GridParams gp{};
  gp.kind = g.kind;
  gp.nv = g.num_views;
  gp.nr = g.num_rows;
  gp.nc = g.num_cols;
  gp.nx = g.num_x;
  gp.ny = g.num_y;
  gp.nz = g.num_z;
  gp.batch = 1;
  gp.hx = (float)g.voxel_width;
  gp.hz = (float)g.voxel_height;
  gp.pw = (float)g.pixel_width;
  gp.ph = (float)g.pixel_height;
  gp.cr = (float)g.center_row;
  gp.cc = (float)g.center_col;
  gp.sdd = (float)g.sdd;
  gp.half_x = 0.5f * (float)g.num_x;
  gp.half_y = 0.5f * (float)g.num_y;
  gp.inv_ph = (float)(1.0 / g.pixel_height);
  gp.hz_over_ph = (float)(g.voxel_height / g.pixel_height);
  gp.e_par = (float)(0.5 * g.voxel_height / g.pixel_height);
  return gp;
}

size_t align_up(size_t n) { return (n + 255) & ~size_t(255); }

int check_run_args(const ctp_plan* plan, const void* in, const void* out, int batch,
                   void* ws, size_t ws_bytes, size_t need) {
  if (!plan) return fail(CTP_ERR_INVALID_ARGUMENT, "plan is null");
  if (!in || !out) return fail(CTP_ERR_INVALID_ARGUMENT, "null data pointer");
  if (batch < 1) return fail(CTP_ERR_INVALID_ARGUMENT, "batch must be >= 1");
  if (in == out) return fail(CTP_ERR_INVALID_ARGUMENT, "input and output must not alias");
  if (ws_bytes < need || (need > 0 && !ws))
    return fail(CTP_ERR_WORKSPACE, "workspace too small: need " + std::to_string(need) + " bytes");
  return CTP_OK;
}

// record an event pair around the projector kernel when timing is requested
struct KernelTimer {
  ctp_plan* p;
  int dir;
  cudaStream_t s;
  bool on;
  KernelTimer(const ctp_plan* plan, int direction, cudaStream_t st, uint32_t flags)
      : p(const_cast<ctp_plan*>(plan)), dir(direction), s(st), on((flags & CTP_FLAG_TIME_KERNEL) != 0) {
    if (!on) return;
    for (int k = 0; k < 2; ++k)
      if (!p->ev[dir][k]) cudaEventCreate(&p->ev[dir][k]);
    cudaEventRecord(p->ev[dir][0], s);
  }
  void stop() {
    if (!on) return;
    cudaEventRecord(p->ev[dir][1], s);
    p->ev_recorded[dir] = true;
  }
};

}  // namespace

extern "C" {

int ctp_abi_version(void) { return CTP_ABI_VERSION; }

const char* ctp_status_string(int status) {
  switch (status) {
    case CTP_OK: return "ok";
    case CTP_ERR_INVALID_ARGUMENT: return "invalid argument";
    case CTP_ERR_UNSUPPORTED_GEOMETRY: return "unsupported geometry";
    case CTP_ERR_SPEC_MISMATCH: return "spec mismatch";
    case CTP_ERR_CUDA: return "CUDA runtime error";
    case CTP_ERR_OUT_OF_MEMORY: return "out of device memory";
    case CTP_ERR_WORKSPACE: return "workspace too small";
    default: return "unknown status";
  }
}

int ctp_last_error(char* buf, size_t buf_bytes) {
  if (!buf || buf_bytes == 0) return CTP_ERR_INVALID_ARGUMENT;
  std::snprintf(buf, buf_bytes, "%s", g_last_error.c_str());
  return CTP_OK;
}

int ctp_plan_create(const ctp_geom* geom, int device, ctp_plan** plan_out) {
  if (!plan_out) return fail(CTP_ERR_INVALID_ARGUMENT, "plan_out is null");
  *plan_out = nullptr;
  int st = validate(geom);
  if (st != CTP_OK) return st;
  DeviceGuard guard(device);
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "select device");
  ctp_plan* p = new (std::nothrow) ctp_plan();
  if (!p) return fail(CTP_ERR_OUT_OF_MEMORY, "host allocation failed");
  p->geom = *geom;
  p->geom.poses = nullptr;
  p->poses.assign(geom->poses, geom->poses + 15 * (size_t)geom->num_views);
  cudaGetDevice(&p->device);
  p->gp = make_grid_params(*geom);
  p->vol_elems = (size_t)geom->num_x * geom->num_y * geom->num_z;
  p->sino_elems = (size_t)geom->num_views * geom->num_rows * geom->num_cols;
  std::vector<ViewCoef> coefs;
  std::vector<ViewAx> axs;
  build_view_coefs(*geom, p->poses.data(), coefs, axs);
  cudaError_t e = cudaMalloc(&p->d_coef, sizeof(ViewCoef) * coefs.size());
  if (e != cudaSuccess) {
    delete p;
    return cuda_fail(e, "cudaMalloc(view coefficients)");
  }
  e = cudaMemcpy(p->d_coef, coefs.data(), sizeof(ViewCoef) * coefs.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&p->d_ax, sizeof(ViewAx) * axs.size());
  if (e == cudaSuccess) e = cudaMemcpy(p->d_ax, axs.data(), sizeof(ViewAx) * axs.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&p->d_pose, sizeof(double) * p->poses.size());
  if (e == cudaSuccess)
    e = cudaMemcpy(p->d_pose, p->poses.data(), sizeof(double) * p->poses.size(), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(p->d_coef);
    if (p->d_ax) cudaFree(p->d_ax);
    if (p->d_pose) cudaFree(p->d_pose);
    delete p;
    return cuda_fail(e, "upload view tables");
  }
  p->sf_ok = sf_supports(geom);
  *plan_out = p;
  return CTP_OK;
}

int ctp_plan_destroy(ctp_plan* plan) {
  if (!plan) return CTP_OK;
  DeviceGuard guard(plan->device);
  if (plan->d_coef) cudaFree(plan->d_coef);
  if (plan->d_ax) cudaFree(plan->d_ax);
  if (plan->d_pose) cudaFree(plan->d_pose);
  for (int d = 0; d < 2; ++d)
    for (int k = 0; k < 2; ++k)
      if (plan->ev[d][k]) cudaEventDestroy(plan->ev[d][k]);
  delete plan;
  return CTP_OK;
}

int ctp_plan_shape(const ctp_plan* plan, int64_t* vol_elems, int64_t* sino_elems) {
  if (!plan) return fail(CTP_ERR_INVALID_ARGUMENT, "plan is null");
  if (vol_elems) *vol_elems = (int64_t)plan->vol_elems;
  if (sino_elems) *sino_elems = (int64_t)plan->sino_elems;
  return CTP_OK;
}

// fan beam (one slice, one detector row) with a batch: batch-on-lanes kernels
static bool use_fan_path(const ctp_plan* plan, int batch, uint32_t flags) {
  return plan->gp.nz == 1 && plan->gp.nr == 1 && batch >= 2 && !(flags & CTP_FLAG_ACCUMULATE);
}

size_t ctp_sf_workspace_bytes(const ctp_plan* plan, int direction, int batch) {
  if (!plan || batch < 1) return 0;
  // a transposed copy of the input: z-contiguous volume / row-contiguous
  // sinogram (3D), batch-innermost input (fan; the fan kernels write the
  // natural output layout directly)
  const size_t per = direction == 0 ? plan->vol_elems : plan->sino_elems;
  return align_up(per * sizeof(float) * (size_t)batch);
}

static int check_sf(const ctp_plan* plan) {
  if (plan && !plan->sf_ok)
    return fail(CTP_ERR_UNSUPPORTED_GEOMETRY,
                "SF-modular needs upright detector panels (colDir.z == 0, rowDir == +z) in every view; "
                "use the Siddon model for tilted panels");
  return CTP_OK;
}

int ctp_sf_forward(const ctp_plan* plan, const float* vol, float* sino, int batch, void* workspace,
                   size_t workspace_bytes, uint32_t flags, void* stream) {
  const size_t need = plan ? ctp_sf_workspace_bytes(plan, 0, batch) : 0;
  int st = check_run_args(plan, vol, sino, batch, workspace, workspace_bytes, need);
  if (st == CTP_OK) st = check_sf(plan);
  if (st != CTP_OK) return st;
  DeviceGuard guard(plan->device);
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "select device");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const GridParams& gp = plan->gp;
  if (use_fan_path(plan, batch, flags)) {
    float* xB = static_cast<float*>(workspace);
    cudaError_t e = ctp::launch_transpose(vol, xB, batch, (int)plan->vol_elems, 1, s);
    if (e != cudaSuccess) return cuda_fail(e, "transpose volume (fan)");
    KernelTimer timer(plan, 0, s, flags);
    e = ctp::launch_forward_fan(gp, plan->d_coef, xB, sino, batch, s);
    timer.stop();
    if (e != cudaSuccess) return cuda_fail(e, "sf_forward_fan_kernel");
    return CTP_OK;
  }
  float* xT = static_cast<float*>(workspace);
  cudaError_t e = ctp::launch_transpose(vol, xT, gp.nz, gp.nx * gp.ny, batch, s);
  if (e != cudaSuccess) return cuda_fail(e, "transpose volume");
  KernelTimer timer(plan, 0, s, flags);
  e = ctp::launch_forward(gp, plan->d_coef, plan->d_ax, xT, sino, batch, (flags & CTP_FLAG_ACCUMULATE) != 0, s);
  timer.stop();
  if (e != cudaSuccess) return cuda_fail(e, "sf_forward_kernel");
  return CTP_OK;
}

int ctp_sf_back(const ctp_plan* plan, const float* sino, float* vol, int batch, void* workspace,
                size_t workspace_bytes, uint32_t flags, void* stream) {
  const size_t need = plan ? ctp_sf_workspace_bytes(plan, 1, batch) : 0;
  int st = check_run_args(plan, sino, vol, batch, workspace, workspace_bytes, need);
  if (st == CTP_OK) st = check_sf(plan);
  if (st != CTP_OK) return st;
  DeviceGuard guard(plan->device);
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "select device");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const GridParams& gp = plan->gp;
  if (use_fan_path(plan, batch, flags)) {
    float* yB = static_cast<float*>(workspace);
    cudaError_t e = ctp::launch_transpose(sino, yB, batch, (int)plan->sino_elems, 1, s);
    if (e != cudaSuccess) return cuda_fail(e, "transpose sinogram (fan)");
    KernelTimer timer(plan, 1, s, flags);
    e = ctp::launch_back_fan(gp, plan->d_coef, yB, vol, batch, s);
    timer.stop();
    if (e != cudaSuccess) return cuda_fail(e, "sf_back_fan_kernel");
    return CTP_OK;
  }
  float* yT = static_cast<float*>(workspace);
  cudaError_t e = ctp::launch_back_input(sino, yT, gp.nr, gp.nc, batch * gp.nv, s);
  if (e != cudaSuccess) return cuda_fail(e, "transpose_segscan_kernel");
  KernelTimer timer(plan, 1, s, flags);
  e = ctp::launch_back(gp, plan->d_coef, plan->d_ax, yT, vol, batch, (flags & CTP_FLAG_ACCUMULATE) != 0, s);
  timer.stop();
  if (e != cudaSuccess) return cuda_fail(e, "sf_back_kernel");
  return CTP_OK;
}

static ctp::SiddonParams siddon_params(const ctp_geom& g, double back) {
  ctp::SiddonParams p;
  p.kind = g.kind;
  p.nv = g.num_views;
  p.nr = g.num_rows;
  p.nc = g.num_cols;
  p.nx = g.num_x;
  p.ny = g.num_y;
  p.nz = g.num_z;
  p.pw = g.pixel_width;
  p.ph = g.pixel_height;
  p.cr = g.center_row;
  p.cc = g.center_col;
  p.sdd = g.sdd;
  p.back = back;
  p.x0 = g.x0;
  p.y0 = g.y0;
  p.z0 = g.z0;
  p.hx = g.voxel_width;
  p.hz = g.voxel_height;
  return p;
}

int ctp_siddon_forward(const ctp_plan* plan, double back, const float* vol, float* sino, int batch,
                       uint32_t flags, void* stream) {
  int st = check_run_args(plan, vol, sino, batch, nullptr, 0, 0);
  if (st != CTP_OK) return st;
  if (!std::isfinite(back)) return fail(CTP_ERR_INVALID_ARGUMENT, "back must be finite");
  DeviceGuard guard(plan->device);
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "select device");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  KernelTimer timer(plan, 0, s, flags);
  cudaError_t e = ctp::launch_siddon_forward(siddon_params(plan->geom, back), plan->d_pose, vol, sino, batch,
                                             (flags & CTP_FLAG_ACCUMULATE) != 0, s);
  timer.stop();
  if (e != cudaSuccess) return cuda_fail(e, "siddon_forward_kernel");
  return CTP_OK;
}

int ctp_siddon_back(const ctp_plan* plan, double back, const float* sino, float* vol, int batch,
                    uint32_t flags, void* stream) {
  int st = check_run_args(plan, sino, vol, batch, nullptr, 0, 0);
  if (st != CTP_OK) return st;
  if (!std::isfinite(back)) return fail(CTP_ERR_INVALID_ARGUMENT, "back must be finite");
  DeviceGuard guard(plan->device);
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "select device");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const ctp::SiddonParams sp = siddon_params(plan->geom, back);
  // stream-ordered scratch for the per-pixel ray table (skipped above 8 GiB:
  // the gather then recomputes each ray)
  const size_t tb = ctp::siddon_ray_table_bytes(sp);
  void* table = nullptr;
  if (tb <= (size_t(8) << 30) && cudaMallocAsync(&table, tb, s) != cudaSuccess) {
    cudaGetLastError();  // clear; fall back to recomputing the rays
    table = nullptr;
  }
  KernelTimer timer(plan, 1, s, flags);
  cudaError_t e = ctp::launch_siddon_back(sp, plan->d_pose, sino, vol, batch, (flags & CTP_FLAG_ACCUMULATE) != 0,
                                          table, s);
  timer.stop();
  if (table) cudaFreeAsync(table, s);
  if (e != cudaSuccess) return cuda_fail(e, "siddon_back_kernel");
  return CTP_OK;
}

int ctp_sf_fbp_back(const ctp_plan* plan, const float* sino, float* vol, int batch, double scale,
                    void* workspace, size_t workspace_bytes, uint32_t flags, void* stream) {
  const size_t need = plan ? ctp_sf_workspace_bytes(plan, 1, batch) : 0;
  int st = check_run_args(plan, sino, vol, batch, workspace, workspace_bytes, need);
  if (st == CTP_OK) st = check_sf(plan);
  if (st != CTP_OK) return st;
  if (!std::isfinite(scale)) return fail(CTP_ERR_INVALID_ARGUMENT, "scale must be finite");
  DeviceGuard guard(plan->device);
  if (guard.err != cudaSuccess) return cuda_fail(guard.err, "select device");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const GridParams& gp = plan->gp;
  // ramp filter fused with the row-contiguous layout change (replaces the
  // back projection's transpose), then the 3D back projection kernel
  float* yT = static_cast<float*>(workspace);
  cudaError_t e = ctp::launch_ramp_rows_T(sino, yT, gp.nr, gp.nc, batch * gp.nv, plan->geom.pixel_width, scale, s);
  if (e != cudaSuccess) return cuda_fail(e, "ramp_rows_T_kernel");
  e = ctp::launch_back_input_inplace(yT, gp.nr, gp.nc, batch * gp.nv, s);
  if (e != cudaSuccess) return cuda_fail(e, "segscan_rows_kernel");
  KernelTimer timer(plan, 1, s, flags);
  e = ctp::launch_back(gp, plan->d_coef, plan->d_ax, yT, vol, batch, (flags & CTP_FLAG_ACCUMULATE) != 0, s);
  timer.stop();
  if (e != cudaSuccess) return cuda_fail(e, "sf_back_kernel (fbp)");
  return CTP_OK;
}

int ctp_plan_kernel_time_ms(const ctp_plan* plan, int direction, float* ms) {
  if (!plan || !ms || direction < 0 || direction > 1)
    return fail(CTP_ERR_INVALID_ARGUMENT, "bad arguments");
  if (!plan->ev_recorded[direction])
    return fail(CTP_ERR_INVALID_ARGUMENT, "no timed launch recorded for this direction");
  DeviceGuard guard(plan->device);
  cudaError_t e = cudaEventSynchronize(plan->ev[direction][1]);
  if (e != cudaSuccess) return cuda_fail(e, "cudaEventSynchronize");
  e = cudaEventElapsedTime(ms, plan->ev[direction][0], plan->ev[direction][1]);
  if (e != cudaSuccess) return cuda_fail(e, "cudaEventElapsedTime");
  return CTP_OK;
}

static int oneshot(const ctp_geom* geom, const float* in, float* out, int batch, void* stream,
                   int direction) {
  ctp_plan* plan = nullptr;
  int st = ctp_plan_create(geom, -1, &plan);
  if (st != CTP_OK) return st;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const size_t need = ctp_sf_workspace_bytes(plan, direction, batch);
  void* ws = nullptr;
  cudaError_t e = cudaMallocAsync(&ws, need, s);
  if (e != cudaSuccess) {
    ctp_plan_destroy(plan);
    return cuda_fail(e, "cudaMallocAsync(workspace)");
  }
  st = direction == 0 ? ctp_sf_forward(plan, in, out, batch, ws, need, 0, stream)
                      : ctp_sf_back(plan, in, out, batch, ws, need, 0, stream);
  cudaFreeAsync(ws, s);
  e = cudaStreamSynchronize(s);
  ctp_plan_destroy(plan);
  if (st != CTP_OK) return st;
  if (e != cudaSuccess) return cuda_fail(e, "stream synchronize");
  return CTP_OK;
}

int ctp_sf_forward_oneshot(const ctp_geom* geom, const float* vol, float* sino, int batch,
                           void* stream) {
  return oneshot(geom, vol, sino, batch, stream, 0);
}

int ctp_sf_back_oneshot(const ctp_geom* geom, const float* sino, float* vol, int batch,
                        void* stream) {
  return oneshot(geom, sino, vol, batch, stream, 1);
}

}  // extern "C"
