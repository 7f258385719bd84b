// sf_common.cuh -- shared host/device definitions of the SF-TR projector pair.
//
// The forward (ray-driven gather) and back (voxel-driven gather) kernels both
// evaluate the separable-footprint coefficient
//
//     a(voxel, view, row, col) = (amp * tt(row)) * ts(col)
//
// of the reference (_kernels.py:555-647 forward, 666-763 back) through the
// functions in this header.  Every floating-point step of the coefficient is
// written with explicit-rounding intrinsics (__fmul_rn, __fadd_rn, __fmaf_rn,
// ...) so that nvcc cannot contract or reassociate it differently in the two
// kernels.  The fan pair shares every operand and is an exact fp32 transpose;
// the 3D pair measures footprint edges from different local origins (the
// forward's band row, the back's table row; see fill_entry / localize_entry)
// and is a transpose to fp32 rounding (explicit-matrix test,
// pkg/tests/test_sf.py:89-111, at 4e-6 of max|A|).
//
// Coordinates.  Geometry is pre-digested on the host in float64 (ctp_plan)
// into per-view affine coefficients over CENTRED GRID-INDEX coordinates
// (X, Y) = (ix + 0.5 - nx/2, iy + 0.5 - ny/2) for voxel centres (corners sit
// at half-integers of that frame).  Detector coordinates are expressed in
// pixel units: column coordinate S = s/pw + cc, row coordinate T = t/ph + cr,
// so detector column c covers [c - 0.5, c + 0.5] and row r covers
// [r - 0.5, r + 0.5].  Keeping magnitudes small (|X|,|Y| <= n/2, |S|,|T| <=
// n_det) holds fp32 rounding of the footprint edges near 1e-5 pixel.
#pragma once

#include <cstdint>

#ifndef __CUDACC__
#define __host__
#define __device__
#define __forceinline__ inline
#endif

namespace ctp {

enum Kind : int { kParallel = 0, kConeFlat = 1, kConeCurved = 2, kModular = 3 };

// Per-view coefficient block (built on the host in f64 by build_view_coefs in
// capi.cu; 32 floats = 128 B, read with broadcast loads).
struct alignas(16) ViewCoef {
  // transverse numerator, affine in (X, Y).  parallel: S itself;
  // flat: r.u with r = p - src at z = 0; curved: r.u (xy only)
  float na, nb, nc;
  // transverse denominator.  flat: r.n (n = u x vax, incl. the z term of
  // _flat_plane_s); curved: r.w (xy only).  parallel: unused
  float da, db, dc;
  float dm;      // flat: centre denominator constant (rcx*nxv + rcy*nyv, no z term)
  float s0;      // column offset (flat: (src-c0).u/pw + cc; curved: cc)
  float g;       // flat: lamnum/pw; curved: sdd/pw
  float lamnum;  // flat: (c0-src).n ; curved: sdd
  float dxa, dya;  // centre offset from the source in mm: xm - sx, ym - sy
  float zc0;       // cone: z of the first slice centre minus source z (mm)
  float ta, tb, tc, tz;  // parallel axial map T = ta + tb X + tc Y + tz iz
  float ux, uy;          // detector transverse axis (split-axis choice, ray setup)
  float wx, wy;          // central ray direction (parallel lxy, curved ax test)
  float xs, ys;          // source in centred grid-index coords
  float xc0, yc0;        // detector reference point c0 in centred grid-index coords
  int cull;              // 1: wedge culling is safe for this view (source outside grid)
  int split_x;           // _sf_subdivide axis decided in f64: |u_x| hx >= |u_y| hx
  float tva;             // modular: ((xm-sx) v_x + (ym-sy) v_y) / ph
  float pad[2];
};
static_assert(sizeof(ViewCoef) == 128, "ViewCoef must stay 128 bytes");

// Per-view float64 axial map (built with ViewCoef in capi.cu).  For a voxel
// column centred at (X, Y) (centred grid-index coords):
//   mag = lam / den,   den = k0 + k1 X + k2 Y      (flat cone, modular, parallel: lam = k0 = 1)
//   mag = lam / rho,   rho = |(k0 + k2 X, k1 + k2 Y)|  (curved cone: k2 = hx)
//   A   = a0 + mag (a1 + a2 X + a3 Y)   row coordinate of slice 0's centre
//   B   = mag bz                        rows per slice (E = B / 2)
// i.e. exactly the axial map of _kernels.py:619-645 (tcen / ph + cr,
// te = mag hz / 2).  The 3D kernels evaluate it in f64 once per (column,
// view) and hand the kernels positions RELATIVE to a local origin, so fp32
// resolves footprint edges to ~1e-5 row even on 1536-row detectors.
struct alignas(16) ViewAx {
  double k0, k1, k2, lam;
  double a0, a1, a2, a3;
  double bz;
  double pad[3];
};
static_assert(sizeof(ViewAx) == 96, "ViewAx layout");

// Launch-invariant scalars.
struct GridParams {
  int kind;
  int nv, nr, nc;
  int nx, ny, nz;
  int batch;
  float hx, hz;        // voxel pitches (mm)
  float pw, ph;        // pixel pitches (mm)
  float cr, cc;        // detector centre (pixels)
  float sdd;
  float half_x, half_y;  // nx/2, ny/2
  float inv_ph;          // 1/ph
  float hz_over_ph;      // hz/ph
  float e_par;           // parallel axial half-width: 0.5*hz/ph
};

// One (sub-)voxel column's footprint in one view.
struct SubFoot {
  float t0, t1, t2, t3;  // sorted transverse breakpoints (column units)
  float A, B, E;         // axial: T(iz) = A + B*iz, half-width E (row units)
  float lxy, a0, a1;     // amp(iz) = lxy * sqrt(1 + (a0 + a1*iz)^2)
  int cl, ch;            // clamped detector-column range (cl > ch: none)
};

#ifdef __CUDACC__

// ---- explicit-rounding helpers (no contraction across kernels) ------------
__device__ __forceinline__ float mul_(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float add_(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub_(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fma_(float a, float b, float c) { return __fmaf_rn(a, b, c); }
__device__ __forceinline__ float div_(float a, float b) { return __fdiv_rn(a, b); }
// hardware sqrt approximation: deterministic, ~1 ulp; amplitude only
__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// packed f32x2 arithmetic (sm_100a FADD2/FMUL2/FFMA2): two independent IEEE
// single-precision operations, so results equal the scalar intrinsics above
__device__ __forceinline__ float2 add2_(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 mul2_(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mul.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 fma2_(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "mov.b64 rc, {%6, %7};\n\tfma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 bc2_(float a) { return make_float2(a, a); }

__device__ __forceinline__ float affine_(float a, float b, float c, float X, float Y) {
  return fma_(c, Y, fma_(b, X, a));
}

// _sort4, _kernels.py:393-405 (same comparator network, branch-free)
__device__ __forceinline__ void sort4f(float& a, float& b, float& c, float& d) {
  float lo, hi;
  lo = fminf(a, b); hi = fmaxf(a, b); a = lo; b = hi;
  lo = fminf(c, d); hi = fmaxf(c, d); c = lo; d = hi;
  lo = fminf(a, c); hi = fmaxf(a, c); a = lo; c = hi;
  lo = fminf(b, d); hi = fmaxf(b, d); b = lo; d = hi;
  lo = fminf(b, c); hi = fmaxf(b, c); b = lo; c = hi;
}

// _trap_cum, _kernels.py:408-420, in column units, branch-free (the setup is
// evaluated lane-parallel over views, so branches would diverge): integral of
// the unit trapezoid (t0..t3) from t0 up to s, as rising + flat + falling parts
//   L = 0.5 (a - t0)^2 / (t1 - t0),              a = clamp(s, t0, t1)
//   M = b - t1,                                  b = clamp(s, t1, t2)
//   R = (c - t2) ((t3 - c) + (t3 - t2)) / (2 (t3 - t2)),  c = clamp(s, t2, t3)
// Degenerate edges (t0 == t1 or t2 == t3) use a zero reciprocal.
struct Trap {
  float t0, t1, t2, t3;
  float i01, i23;  // 0.5/(t1-t0), 0.5/(t3-t2) (0 when degenerate)
};
__device__ __forceinline__ Trap make_trap(const SubFoot& f) {
  Trap p;
  p.t0 = f.t0; p.t1 = f.t1; p.t2 = f.t2; p.t3 = f.t3;
  const float w01 = sub_(f.t1, f.t0), w23 = sub_(f.t3, f.t2);
  p.i01 = w01 > 0.0f ? div_(0.5f, w01) : 0.0f;
  p.i23 = w23 > 0.0f ? div_(0.5f, w23) : 0.0f;
  return p;
}
__device__ __forceinline__ float clampf_(float x, float lo, float hi) {
  return fminf(fmaxf(x, lo), hi);
}
__device__ __forceinline__ float trap_cum(const Trap& p, float s) {
  const float a = sub_(clampf_(s, p.t0, p.t1), p.t0);
  const float b = sub_(clampf_(s, p.t1, p.t2), p.t1);
  const float c = clampf_(s, p.t2, p.t3);
  const float L = mul_(mul_(a, a), p.i01);
  const float R = mul_(mul_(sub_(c, p.t2), add_(sub_(p.t3, c), sub_(p.t3, p.t2))), p.i23);
  return add_(add_(L, b), R);
}

// Column weight T_s(col) = F(col+0.5) - F(col-0.5) (the /pw of
// _kernels.py:610-614 is implicit in column units).
__device__ __forceinline__ float col_weight(const Trap& p, int col) {
  const float c = (float)col;
  return sub_(trap_cum(p, add_(c, 0.5f)), trap_cum(p, sub_(c, 0.5f)));
}

// Column weights of NW consecutive detector columns c_first.. : NW+1 shared
// boundary evaluations of the trapezoid integral.  ts(c) = F(c+.5) - F(c-.5)
// with exactly the same F values wherever a boundary is shared, so any caller
// (back: footprint columns, forward: tile columns) gets bitwise equal weights.
template <int NW>
__device__ __forceinline__ void col_weights(const Trap& p, int c_first, float (&ts)[NW]) {
  float prev = trap_cum(p, sub_((float)c_first, 0.5f));
#pragma unroll
  for (int k = 0; k < NW; ++k) {
    const float cur = trap_cum(p, add_((float)(c_first + k), 0.5f));
    ts[k] = sub_(cur, prev);
    prev = cur;
  }
}

// Axial map (_kernels.py:619-645) in row units: slice iz spans
// [T - E, T + E] with T = A + B iz; its weight in row r is the overlap with
// [r - 0.5, r + 0.5] written as a difference of clamped boundaries,
//   tt(r) = clamp(r + 0.5, lo, hi) - clamp(r - 0.5, lo, hi),
// which both kernels evaluate identically (r +- 0.5 is exact in fp32).
__device__ __forceinline__ float row_center(const SubFoot& f, int iz) {
  return fma_(f.B, (float)iz, f.A);
}
__device__ __forceinline__ float row_overlap(float lo, float hi, int row) {
  const float r = (float)row;
  return sub_(clampf_(add_(r, 0.5f), lo, hi), clampf_(sub_(r, 0.5f), lo, hi));
}
// First row whose interval can overlap [lo, hi]: min{ r : r + 0.5 > lo }
// = floor(lo - 0.5) + 1.  For |lo| < 2^22 the subtraction lo - 0.5 is exact
// in fp32 (both operands are multiples of ulp(lo) <= 0.5, Sterbenz below 1),
// so rows below first_row have exactly zero overlap.  row_floor returns
// floor(lo - 0.5) = r0 - 1 as an integer-valued float; the boundaries of row
// r0 + k are then row_floor + 0.5 + k and row_floor + 1.5 + k (exact).
__device__ __forceinline__ float row_floor(float lo) { return floorf(sub_(lo, 0.5f)); }
__device__ __forceinline__ int first_row(float lo) { return (int)row_floor(lo) + 1; }
// Rows a slice of axial height 2E = B can touch, counted from first_row
// (with a 1e-3 margin against fp32 rounding of lo / hi).
__device__ __forceinline__ int rows_per_slice(float B) { return (int)(B + 1.001f) + 1; }

// SF amplitude (_sf_amplitude, _kernels.py:529-539): lxy / cos(axial tilt)
__device__ __forceinline__ float amplitude(const SubFoot& f, int iz) {
  const float q = fma_(f.a1, (float)iz, f.a0);
  return mul_(f.lxy, sqrt_approx(fma_(q, q, 1.0f)));
}

// _sf_transverse (_kernels.py:441-526) + axial setup for one sub-voxel whose
// centre is (X, Y) (centred grid-index coords) with half-widths (hxi, hyi) in
// index units.  Returns false on the reference's ok=False paths.
__device__ __forceinline__ bool sub_footprint(const ViewCoef& v, const GridParams& gp,
                                              float X, float Y, float hxi, float hyi,
                                              SubFoot& f) {
  const float xa = sub_(X, hxi), xb = add_(X, hxi);
  const float ya = sub_(Y, hyi), yb = add_(Y, hyi);
  const float hxw = mul_(hxi, gp.hx), hyw = mul_(hyi, gp.hx);  // world half-widths
  float s0, s1, s2, s3, dxn, dyn;
  if (gp.kind == kParallel) {
    s0 = affine_(v.na, v.nb, v.nc, xa, ya);
    s1 = affine_(v.na, v.nb, v.nc, xb, ya);
    s2 = affine_(v.na, v.nb, v.nc, xa, yb);
    s3 = affine_(v.na, v.nb, v.nc, xb, yb);
    dxn = v.wx;
    dyn = v.wy;
    f.A = affine_(v.ta, v.tb, v.tc, X, Y);
    f.B = v.tz;
    f.E = gp.e_par;
    f.a0 = 0.0f;
    f.a1 = 0.0f;
  } else {
    const float dx = fma_(gp.hx, X, v.dxa), dy = fma_(gp.hx, Y, v.dya);
    const float rho = __fsqrt_rn(fma_(dx, dx, mul_(dy, dy)));
    if (!(rho >= 1e-9f)) return false;
    float mag;
    if (gp.kind == kConeCurved) {
      if (!(fma_(dx, v.wx, mul_(dy, v.wy)) > 0.0f)) return false;
      mag = div_(gp.sdd, rho);
      s0 = fma_(v.g, atan2f(affine_(v.na, v.nb, v.nc, xa, ya), affine_(v.da, v.db, v.dc, xa, ya)), v.s0);
      s1 = fma_(v.g, atan2f(affine_(v.na, v.nb, v.nc, xb, ya), affine_(v.da, v.db, v.dc, xb, ya)), v.s0);
      s2 = fma_(v.g, atan2f(affine_(v.na, v.nb, v.nc, xa, yb), affine_(v.da, v.db, v.dc, xa, yb)), v.s0);
      s3 = fma_(v.g, atan2f(affine_(v.na, v.nb, v.nc, xb, yb), affine_(v.da, v.db, v.dc, xb, yb)), v.s0);
    } else {
      // flat panel: ray/plane intersection (_flat_plane_s, _kernels.py:423-438)
      float d[4], n[4];
      d[0] = affine_(v.da, v.db, v.dc, xa, ya); n[0] = affine_(v.na, v.nb, v.nc, xa, ya);
      d[1] = affine_(v.da, v.db, v.dc, xb, ya); n[1] = affine_(v.na, v.nb, v.nc, xb, ya);
      d[2] = affine_(v.da, v.db, v.dc, xa, yb); n[2] = affine_(v.na, v.nb, v.nc, xa, yb);
      d[3] = affine_(v.da, v.db, v.dc, xb, yb); n[3] = affine_(v.na, v.nb, v.nc, xb, yb);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (!(fabsf(d[k]) > 1e-12f)) return false;
        if (!(div_(v.lamnum, d[k]) > 0.0f)) return false;
      }
      s0 = fma_(v.g, div_(n[0], d[0]), v.s0);
      s1 = fma_(v.g, div_(n[1], d[1]), v.s0);
      s2 = fma_(v.g, div_(n[2], d[2]), v.s0);
      s3 = fma_(v.g, div_(n[3], d[3]), v.s0);
      const float den = affine_(v.dm, v.db, v.dc, X, Y);
      if (!(fabsf(den) > 1e-12f)) return false;
      mag = div_(v.lamnum, den);
      if (!(mag > 0.0f)) return false;
    }
    dxn = div_(dx, rho);
    dyn = div_(dy, rho);
    if (gp.kind == kModular) {
      // modular (extension): row coordinate of the column centre
      // line t(z) = (src-c0).v + mag ((c-src)_xy . v_xy + v_z (z - src_z)),
      // affine in z; ta = (src-c0).v/ph + cr, tb/tc/tva the xy part, tz = v_z
      const float txy = affine_(v.tva, v.tb, v.tc, X, Y);
      const float bm = mul_(mag, mul_(v.tz, gp.hz_over_ph));
      f.B = bm;
      f.E = mul_(0.5f, bm);
      f.A = fma_(mag, fma_(mul_(v.tz, gp.inv_ph), v.zc0, txy), v.ta);
    } else {
      // axial: tcen = mag*(cz - src_z)  (_kernels.py:626-628), in row units
      const float bm = mul_(mag, gp.hz_over_ph);
      f.B = bm;
      f.E = mul_(0.5f, bm);
      f.A = fma_(mul_(mag, v.zc0), gp.inv_ph, gp.cr);
    }
    f.a0 = div_(v.zc0, rho);
    f.a1 = div_(gp.hz, rho);
  }
  sort4f(s0, s1, s2, s3);
  f.t0 = s0; f.t1 = s1; f.t2 = s2; f.t3 = s3;
  const float big = 1.0e30f;
  const float la = fabsf(dxn) > 1e-12f ? div_(mul_(2.0f, hxw), fabsf(dxn)) : big;
  const float lb = fabsf(dyn) > 1e-12f ? div_(mul_(2.0f, hyw), fabsf(dyn)) : big;
  f.lxy = fminf(la, lb);
  int cl = (int)ceilf(sub_(s0, 0.5f));
  int ch = (int)floorf(add_(s3, 0.5f));
  f.cl = cl < 0 ? 0 : cl;
  f.ch = ch > gp.nc - 1 ? gp.nc - 1 : ch;
  return true;
}

// Full voxel column (ix, iy) in one view, with the >8-column split of
// _sf_subdivide (_kernels.py:542-552) and the sub-voxel loop of
// _kernels.py:582-601.  Returns a bit mask of valid sub-footprints:
// 1 = s0 only (no split), bits 0/1 = halves of a split voxel (in the
// reference's sub order), 0 = the voxel contributes nothing in this view.
__device__ __forceinline__ int column_footprint(const ViewCoef& v, const GridParams& gp,
                                                int ix, int iy, SubFoot& s0, SubFoot& s1) {
  const float X = sub_((float)ix + 0.5f, gp.half_x);
  const float Y = sub_((float)iy + 0.5f, gp.half_y);
  if (!sub_footprint(v, gp, X, Y, 0.5f, 0.5f, s0)) return 0;
  if (!(sub_(s0.t3, s0.t0) > 8.0f)) return 1;
  const bool along_x = v.split_x != 0;
  const float hxi = along_x ? 0.25f : 0.5f, hyi = along_x ? 0.5f : 0.25f;
  const float X0 = along_x ? sub_(X, 0.25f) : X, Y0 = along_x ? Y : sub_(Y, 0.25f);
  const float X1 = along_x ? add_(X, 0.25f) : X, Y1 = along_x ? Y : add_(Y, 0.25f);
  int mask = 0;
  if (sub_footprint(v, gp, X0, Y0, hxi, hyi, s0)) mask |= 1;
  if (sub_footprint(v, gp, X1, Y1, hxi, hyi, s1)) mask |= 2;
  return mask;
}

// column_footprint plus the (sub-)voxel centres and a split flag (bit 2 of
// the returned mask) for the 3D kernels, which evaluate the axial map of
// each sub-footprint in f64 at its own centre.
__device__ __forceinline__ int column_subs(const ViewCoef& v, const GridParams& gp, int ix, int iy,
                                           SubFoot& s0, SubFoot& s1, float2& c0, float2& c1) {
  const float X = sub_((float)ix + 0.5f, gp.half_x);
  const float Y = sub_((float)iy + 0.5f, gp.half_y);
  c0 = make_float2(X, Y);
  c1 = c0;
  if (!sub_footprint(v, gp, X, Y, 0.5f, 0.5f, s0)) return 0;
  if (!(sub_(s0.t3, s0.t0) > 8.0f)) return 1;
  const bool along_x = v.split_x != 0;
  const float hxi = along_x ? 0.25f : 0.5f, hyi = along_x ? 0.5f : 0.25f;
  c0 = along_x ? make_float2(sub_(X, 0.25f), Y) : make_float2(X, sub_(Y, 0.25f));
  c1 = along_x ? make_float2(add_(X, 0.25f), Y) : make_float2(X, add_(Y, 0.25f));
  int mask = 4;
  if (sub_footprint(v, gp, c0.x, c0.y, hxi, hyi, s0)) mask |= 1;
  if (sub_footprint(v, gp, c1.x, c1.y, hxi, hyi, s1)) mask |= 2;
  return mask;
}

// 1/d to f64 precision without a full DDIV: fp32 reciprocal (~2^-23) and
// two Newton steps in f64 (2^-46, then ~2^-52)
__device__ __forceinline__ double rcp64(double d) {
  double r = (double)__frcp_rn((float)d);
  r = fma(r, fma(-d, r, 1.0), r);
  return fma(r, fma(-d, r, 1.0), r);
}

// f64 axial map of ViewAx at (X, Y): row coordinate A of slice 0's centre and
// rows per slice B.
__device__ __forceinline__ void axial64(const ViewAx& a, int kind, double X, double Y, double& A, double& B) {
  double mag;
  if (kind == kConeCurved) {
    const double dx = fma(a.k2, X, a.k0), dy = fma(a.k2, Y, a.k1);
    mag = a.lam * rcp64(sqrt(fma(dx, dx, dy * dy)));
  } else {
    mag = a.lam * rcp64(fma(a.k2, Y, fma(a.k1, X, a.k0)));
  }
  A = fma(mag, fma(a.a3, Y, fma(a.a2, X, a.a1)), a.a0);
  B = mag * a.bz;
}

// ---- forward-kernel helpers shared by the 3D and fan forward kernels ----
// boundary ray of the tile edge at column coordinate S (centred grid-index coords)
__device__ __forceinline__ void edge_ray(const ViewCoef& vc, const GridParams& gp, float S,
                                         float& px, float& py, float& dx, float& dy) {
  const float s_mm = (S - gp.cc) * gp.pw;  // transverse detector coordinate (mm)
  if (gp.kind == kConeCurved) {
    const float th = s_mm / gp.sdd;
    float sn, cs;
    sincosf(th, &sn, &cs);
    px = vc.xs; py = vc.ys;
    dx = cs * vc.wx + sn * vc.ux;
    dy = cs * vc.wy + sn * vc.uy;
    return;
  }
  if (gp.kind == kModular) {
    // line {S(X, Y) = S} at the reference height: g num - (S - s0) den = 0
    const float kk = S - vc.s0;
    const float al = vc.g * vc.nb - kk * vc.db, be = vc.g * vc.nc - kk * vc.dc;
    const float ga = vc.g * vc.na - kk * vc.da;
    const float n2 = al * al + be * be;
    px = -ga * al / n2;
    py = -ga * be / n2;
    dx = be;
    dy = -al;
    return;
  }
  const float k = s_mm / gp.hx;
  px = vc.xc0 + k * vc.ux;
  py = vc.yc0 + k * vc.uy;
  if (gp.kind == kParallel) {
    dx = vc.wx; dy = vc.wy;
  } else {
    dx = px - vc.xs; dy = py - vc.ys;
  }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
// 16-byte copy of which only the first `bytes` (0..16) are read; the rest of
// the destination is zero-filled
__device__ __forceinline__ void cp_async16_zfill(void* smem, const void* gmem, unsigned bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ int warp_incl_scan(int v, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int n = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += n;
  }
  return v;
}

#endif  // __CUDACC__

}  // namespace ctp
