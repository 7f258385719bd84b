// siddon_kernels.cu -- sm_100a kernels of the Siddon (exact ray-voxel line
// length) projector pair, in float64 like the reference.
//
//   siddon_forward_kernel : one thread per detector sample: the ray through the
//                           pixel centre (_sample_ray, _kernels.py:21-58) is
//                           traced through the grid with merged plane
//                           crossings, each interval attributed to the voxel
//                           holding its midpoint (_siddon_trace, _kernels.py:82-188,
//                           siddon_forward_kernel, _kernels.py:191-208).
//   siddon_back_kernel    : one thread per voxel: for every view, the detector
//                           window bounded by the projections of the voxel's 8
//                           corners (_project_center, _kernels.py:224-279), and
//                           for each pixel in it the exact ray/box clip length
//                           times y (_ray_box_len, _kernels.py:211-221,
//                           siddon_back_kernel, _kernels.py:282-387).
//
// Every floating-point step restates the reference's float64 expression in
// the same order; this file is compiled with -fmad=false so nvcc does not
// contract a*b+c (numba does not either), and double division / sqrt are
// IEEE round-to-nearest.  The forward and back computations of one
// ray/voxel pair therefore agree with the reference's (and with each other)
// to float64 rounding, and the f32 outputs match the reference's.
#include <cuda_runtime.h>

#include <cstdint>

#include "sf_launch.h"

namespace ctp {

namespace {

constexpr double kEpsDir = 1e-12;  // _EPS_DIR
constexpr double kEpsT = 1e-12;    // _EPS_T
constexpr double kInf = 1.0e300;

// per-view pose block: src[0..2], c0[3..5], u[6..8], vax[9..11], w[12..14]
struct Ray {
  double ox, oy, oz, dx, dy, dz;
};

__device__ __forceinline__ Ray sample_ray(const SiddonParams& p, const double* __restrict__ P, int row,
                                          int col) {
  const double s = (col - p.cc) * p.pw;
  const double t = (row - p.cr) * p.ph;
  const double* src = P;
  const double* c0 = P + 3;
  const double* u = P + 6;
  const double* vax = P + 9;
  const double* w = P + 12;
  Ray r;
  if (p.kind == 0) {
    const double px = c0[0] + s * u[0] + t * vax[0];
    const double py = c0[1] + s * u[1] + t * vax[1];
    const double pz = c0[2] + s * u[2] + t * vax[2];
    r.ox = px - p.back * w[0];
    r.oy = py - p.back * w[1];
    r.oz = pz - p.back * w[2];
    r.dx = w[0];
    r.dy = w[1];
    r.dz = w[2];
    return r;
  }
  double px, py, pz;
  if (p.kind == 2) {
    const double al = s / p.sdd;
    const double ca = cos(al), sa = sin(al);
    px = src[0] + p.sdd * (ca * w[0] + sa * u[0]) + t * vax[0];
    py = src[1] + p.sdd * (ca * w[1] + sa * u[1]) + t * vax[1];
    pz = src[2] + p.sdd * (ca * w[2] + sa * u[2]) + t * vax[2];
  } else {
    px = c0[0] + s * u[0] + t * vax[0];
    py = c0[1] + s * u[1] + t * vax[1];
    pz = c0[2] + s * u[2] + t * vax[2];
  }
  const double dx = px - src[0], dy = py - src[1], dz = pz - src[2];
  const double nrm = sqrt(dx * dx + dy * dy + dz * dz);
  r.ox = src[0];
  r.oy = src[1];
  r.oz = src[2];
  r.dx = dx / nrm;
  r.dy = dy / nrm;
  r.dz = dz / nrm;
  return r;
}

// _slab_clip: clip [tmin, tmax] to lo <= o + t d < hi along one axis
__device__ __forceinline__ void slab_clip(double o, double d, double lo, double hi, double& tmin,
                                          double& tmax, bool& ok) {
  if (fabs(d) > kEpsDir) {
    double t1 = (lo - o) / d;
    double t2 = (hi - o) / d;
    if (t1 > t2) {
      const double tt = t1;
      t1 = t2;
      t2 = tt;
    }
    if (t1 > tmin) tmin = t1;
    if (t2 < tmax) tmax = t2;
  } else if (o < lo || o >= hi) {
    ok = false;  // half-open [lo, hi), as the traversal's floor() convention
  }
}

// next plane crossing after tmin along one axis, and the step between crossings
__device__ __forceinline__ void first_crossing(double o, double d, double a0, double h, double tmin,
                                               double& tn, double& st) {
  tn = kInf;
  st = kInf;
  if (fabs(d) > kEpsDir) {
    st = h / fabs(d);
    const double pa = o + tmin * d;
    const double k = floor((pa - a0) / h);
    tn = d > 0.0 ? (a0 + (k + 1.0) * h - o) / d : (a0 + k * h - o) / d;
    while (tn <= tmin) tn += st;
  }
}

// fixed cell index of an axis the ray does not move along (-1 if it moves)
__device__ __forceinline__ int still_index(double o, double d, double a0, double h) {
  if (fabs(d) > kEpsDir) return -1;
  int i = (int)floor((o - a0) / h);
  while (o < a0 + i * h) --i;
  while (o >= a0 + (i + 1) * h) ++i;
  return i;
}

__device__ double siddon_trace(const float* __restrict__ vol, const Ray& r, const SiddonParams& p) {
  const double xhi = p.x0 + p.nx * p.hx, yhi = p.y0 + p.ny * p.hx, zhi = p.z0 + p.nz * p.hz;
  double tmin = -1.0e300, tmax = 1.0e300;
  bool ok = true;
  slab_clip(r.ox, r.dx, p.x0, xhi, tmin, tmax, ok);
  slab_clip(r.oy, r.dy, p.y0, yhi, tmin, tmax, ok);
  slab_clip(r.oz, r.dz, p.z0, zhi, tmin, tmax, ok);
  if (!ok || tmax - tmin < kEpsT) return 0.0;
  double txn, stx, tyn, sty, tzn, stz;
  first_crossing(r.ox, r.dx, p.x0, p.hx, tmin, txn, stx);
  first_crossing(r.oy, r.dy, p.y0, p.hx, tmin, tyn, sty);
  first_crossing(r.oz, r.dz, p.z0, p.hz, tmin, tzn, stz);
  const int ix0 = still_index(r.ox, r.dx, p.x0, p.hx);
  const int iy0 = still_index(r.oy, r.dy, p.y0, p.hx);
  const int iz0 = still_index(r.oz, r.dz, p.z0, p.hz);
  const size_t plane = (size_t)p.nx * p.ny;
  double total = 0.0;
  double tcur = tmin;
  while (tcur < tmax - kEpsT) {
    double tn = txn;
    if (tyn < tn) tn = tyn;
    if (tzn < tn) tn = tzn;
    if (tn > tmax) tn = tmax;
    if (tn > tcur + kEpsT) {
      const double tm = 0.5 * (tcur + tn);
      const int ix = ix0 >= 0 ? ix0 : (int)floor((r.ox + tm * r.dx - p.x0) / p.hx);
      const int iy = iy0 >= 0 ? iy0 : (int)floor((r.oy + tm * r.dy - p.y0) / p.hx);
      const int iz = iz0 >= 0 ? iz0 : (int)floor((r.oz + tm * r.dz - p.z0) / p.hz);
      if (0 <= ix && ix < p.nx && 0 <= iy && iy < p.ny && 0 <= iz && iz < p.nz)
        total += (tn - tcur) * (double)__ldg(vol + (size_t)iz * plane + (size_t)iy * p.nx + ix);
    }
    tcur = tn;
    if (txn <= tn + kEpsT) txn += stx;
    if (tyn <= tn + kEpsT) tyn += sty;
    if (tzn <= tn + kEpsT) tzn += stz;
  }
  return total;
}

__device__ __forceinline__ double ray_box_len(const Ray& r, double xlo, double xhi, double ylo, double yhi,
                                              double zlo, double zhi) {
  double tmin = -1.0e300, tmax = 1.0e300;
  bool ok = true;
  slab_clip(r.ox, r.dx, xlo, xhi, tmin, tmax, ok);
  slab_clip(r.oy, r.dy, ylo, yhi, tmin, tmax, ok);
  slab_clip(r.oz, r.dz, zlo, zhi, tmin, tmax, ok);
  if (!ok || tmax <= tmin) return 0.0;
  return tmax - tmin;
}

// _project_center: detector (s, t) of the line src -> (px, py, pz); false when
// degenerate (the caller then scans the whole detector)
__device__ __forceinline__ bool project_center(const SiddonParams& p, const double* __restrict__ P, double px,
                                               double py, double pz, double& s, double& t) {
  const double* src = P;
  const double* c0 = P + 3;
  const double* u = P + 6;
  const double* vax = P + 9;
  const double* w = P + 12;
  if (p.kind == 0) {
    s = (px - c0[0]) * u[0] + (py - c0[1]) * u[1] + (pz - c0[2]) * u[2];
    t = (px - c0[0]) * vax[0] + (py - c0[1]) * vax[1] + (pz - c0[2]) * vax[2];
    return true;
  }
  const double rx = px - src[0], ry = py - src[1], rz = pz - src[2];
  if (p.kind == 2) {
    const double a = rx * w[0] + ry * w[1] + rz * w[2];
    const double b = rx * u[0] + ry * u[1] + rz * u[2];
    const double rho = sqrt(a * a + b * b);
    if (rho < 1e-9 || a <= 0.0) return false;
    const double zz = rx * vax[0] + ry * vax[1] + rz * vax[2];
    const double mag = p.sdd / rho;
    s = p.sdd * atan2(b, a);
    t = zz * mag;
    return true;
  }
  const double nxv = u[1] * vax[2] - u[2] * vax[1];
  const double nyv = u[2] * vax[0] - u[0] * vax[2];
  const double nzv = u[0] * vax[1] - u[1] * vax[0];
  const double lamnum = (c0[0] - src[0]) * nxv + (c0[1] - src[1]) * nyv + (c0[2] - src[2]) * nzv;
  const double den = rx * nxv + ry * nyv + rz * nzv;
  if (fabs(den) < 1e-12 * (fabs(lamnum) + 1.0)) return false;
  const double lam = lamnum / den;
  if (lam <= 0.0) return false;
  const double qx = src[0] + lam * rx - c0[0];
  const double qy = src[1] + lam * ry - c0[1];
  const double qz = src[2] + lam * rz - c0[2];
  s = qx * u[0] + qy * u[1] + qz * u[2];
  t = qx * vax[0] + qy * vax[1] + qz * vax[2];
  return true;
}

#ifndef CTP_SDF_MINB
#define CTP_SDF_MINB 4
#endif
__global__ void __launch_bounds__(256, CTP_SDF_MINB) siddon_forward_kernel(SiddonParams p, const double* __restrict__ poses,
                                                             const float* __restrict__ vol,
                                                             float* __restrict__ sino, int accumulate) {
  const long long nray = (long long)p.nv * p.nr * p.nc;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nray) return;
  const int b = blockIdx.y;
  const int view = (int)(idx / ((long long)p.nr * p.nc));
  const long long rem = idx - (long long)view * p.nr * p.nc;
  const int row = (int)(rem / p.nc);
  const int col = (int)(rem - (long long)row * p.nc);
  const Ray r = sample_ray(p, poses + 15 * view, row, col);
  const float* vb = vol + (size_t)b * p.nx * p.ny * p.nz;
  const float val = (float)siddon_trace(vb, r, p);
  float* o = sino + (size_t)b * nray + idx;
  *o = accumulate ? *o + val : val;
}

// ray table for the back projector: rays[(view*nr + row)*nc + col] = the
// same Ray sample_ray returns (bitwise), so the gather need not recompute the
// normalisation (sqrt + 3 divisions) for each of its ~20 candidate pixels
__global__ void __launch_bounds__(256) siddon_rays_kernel(SiddonParams p, const double* __restrict__ poses,
                                                          Ray* __restrict__ rays) {
  const long long nray = (long long)p.nv * p.nr * p.nc;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nray) return;
  const int view = (int)(idx / ((long long)p.nr * p.nc));
  const long long rem = idx - (long long)view * p.nr * p.nc;
  const int row = (int)(rem / p.nc);
  const int col = (int)(rem - (long long)row * p.nc);
  rays[idx] = sample_ray(p, poses + 15 * view, row, col);
}

#ifndef CTP_SD_MINB
#define CTP_SD_MINB 4  // 64 registers: occupancy hides the ray-table and division latency
#endif
template <bool TABLE>
__global__ void __launch_bounds__(256, CTP_SD_MINB) siddon_back_kernel(SiddonParams p, const double* __restrict__ poses,
                                                          const Ray* __restrict__ rays,
                                                          const float* __restrict__ sino,
                                                          float* __restrict__ vol, int accumulate) {
  const long long nvox = (long long)p.nx * p.ny * p.nz;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nvox) return;
  const int b = blockIdx.y;
  const int iz = (int)(idx / ((long long)p.nx * p.ny));
  const long long rem = idx - (long long)iz * p.nx * p.ny;
  const int iy = (int)(rem / p.nx);
  const int ix = (int)(rem - (long long)iy * p.nx);
  const double xlo = p.x0 + ix * p.hx, ylo = p.y0 + iy * p.hx, zlo = p.z0 + iz * p.hz;
  const double xhi = xlo + p.hx, yhi = ylo + p.hx, zhi = zlo + p.hz;
  const double cx = xlo + 0.5 * p.hx, cy = ylo + 0.5 * p.hx, cz = zlo + 0.5 * p.hz;
  const double rad2 = (0.5 * p.hx * p.hx + 0.25 * p.hz * p.hz) * (1.0 + 1e-6) + 1e-12;  // (half-diagonal)^2
  const float* yb = sino + (size_t)b * p.nv * p.nr * p.nc;
  double acc = 0.0;
  for (int view = 0; view < p.nv; ++view) {
    const double* P = poses + 15 * view;
    // the rays hitting this convex box lie in the detector shadow of its corners
    double smin = 1.0e300, smax = -1.0e300, tmin = 1.0e300, tmax = -1.0e300;
    bool degen = false;
    for (int corner = 0; corner < 8; ++corner) {
      const double pcx = (corner & 1) ? xlo + p.hx : xlo;
      const double pcy = (corner & 2) ? ylo + p.hx : ylo;
      const double pcz = (corner & 4) ? zlo + p.hz : zlo;
      double s, t;
      if (!project_center(p, P, pcx, pcy, pcz, s, t)) {
        degen = true;
        break;
      }
      if (s < smin) smin = s;
      if (s > smax) smax = s;
      if (t < tmin) tmin = t;
      if (t > tmax) tmax = t;
    }
    int r0 = 0, r1 = p.nr - 1, cl = 0, ch = p.nc - 1;
    if (!degen) {
      cl = max((int)ceil(smin / p.pw + p.cc - 0.5) - 1, 0);
      ch = min((int)floor(smax / p.pw + p.cc + 0.5) + 1, p.nc - 1);
      r0 = max((int)ceil(tmin / p.ph + p.cr - 0.5) - 1, 0);
      r1 = min((int)floor(tmax / p.ph + p.cr + 0.5) + 1, p.nr - 1);
    }
    const float* yv = yb + (size_t)view * p.nr * p.nc;
    const Ray* rv = rays + (size_t)view * p.nr * p.nc;
    for (int row = r0; row <= r1; ++row) {
      for (int col = cl; col <= ch; ++col) {
        const Ray r = TABLE ? rv[(size_t)row * p.nc + col] : sample_ray(p, P, row, col);
        // a ray that meets the box passes within its half-diagonal of the
        // centre; rays clearly farther (the window's padding) contribute an
        // exact 0 and skip the clip (unit directions; the margin dwarfs the
        // rounding of dist2)
        const double vx = cx - r.ox, vy = cy - r.oy, vz = cz - r.oz;
        const double pr = vx * r.dx + vy * r.dy + vz * r.dz;
        const double dist2 = vx * vx + vy * vy + vz * vz - pr * pr;
        if (dist2 > rad2) continue;
        const double ln = ray_box_len(r, xlo, xhi, ylo, yhi, zlo, zhi);
        if (ln > 0.0) acc += ln * (double)__ldg(yv + (size_t)row * p.nc + col);
      }
    }
  }
  float* o = vol + (size_t)b * nvox + idx;
  const float val = (float)acc;
  *o = accumulate ? *o + val : val;
}

}  // namespace

cudaError_t launch_siddon_forward(const SiddonParams& p, const double* poses, const float* vol, float* sino,
                                  int batch, bool accumulate, cudaStream_t st) {
  const long long nray = (long long)p.nv * p.nr * p.nc;
  for (int b0 = 0; b0 < batch; b0 += 65535) {
    const int nb = batch - b0 < 65535 ? batch - b0 : 65535;
    const dim3 grid((unsigned)((nray + 255) / 256), nb);
    siddon_forward_kernel<<<grid, 256, 0, st>>>(p, poses, vol + (size_t)b0 * p.nx * p.ny * p.nz,
                                                sino + (size_t)b0 * nray, accumulate ? 1 : 0);
  }
  return cudaGetLastError();
}

size_t siddon_ray_table_bytes(const SiddonParams& p) {
  return sizeof(Ray) * (size_t)p.nv * p.nr * p.nc;
}

cudaError_t launch_siddon_back(const SiddonParams& p, const double* poses, const float* sino, float* vol,
                               int batch, bool accumulate, void* ray_table, cudaStream_t st) {
  const long long nvox = (long long)p.nx * p.ny * p.nz;
  Ray* rays = static_cast<Ray*>(ray_table);
  if (rays) {
    const long long nray = (long long)p.nv * p.nr * p.nc;
    siddon_rays_kernel<<<(unsigned)((nray + 255) / 256), 256, 0, st>>>(p, poses, rays);
  }
  for (int b0 = 0; b0 < batch; b0 += 65535) {
    const int nb = batch - b0 < 65535 ? batch - b0 : 65535;
    const dim3 grid((unsigned)((nvox + 255) / 256), nb);
    const float* sb = sino + (size_t)b0 * p.nv * p.nr * p.nc;
    float* vb = vol + (size_t)b0 * nvox;
    if (rays)
      siddon_back_kernel<true><<<grid, 256, 0, st>>>(p, poses, rays, sb, vb, accumulate ? 1 : 0);
    else
      siddon_back_kernel<false><<<grid, 256, 0, st>>>(p, poses, nullptr, sb, vb, accumulate ? 1 : 0);
  }
  return cudaGetLastError();
}

}  // namespace ctp
