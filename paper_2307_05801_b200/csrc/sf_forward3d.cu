// sf_forward3d.cu -- 3D forward projection y = A x of the SF-TR pair
// (parallel, cone flat/curved, SF-modular), ray-driven GATHER (reference:
// sf_forward_kernel -> _sf_view_accumulate, _kernels.py:555-663).
//
// Integral formulation.  For one voxel column in one view the axial
// footprints of consecutive slices tile the detector column: slice j spans
// rows [Lo + B j, Lo + B (j + 1)) (row units, B = mag hz / ph), so the
// column's contribution to detector row r is
//
//   P(r) = sum_j overlap(slice j, row r) amp_j x_j = B (Fn(u(r + 1/2)) - Fn(u(r - 1/2))),
//   u(t) = (t - Lo) / B,   Fn(u) = G_k + (u - k) xa_k,   k = floor(u),
//
// with xa_j = amp_j x_j and G_k = sum_{i<k} xa_i.  The reference sums the
// 2-3 overlapping slices of each row (_kernels.py:619-647); here the warp
// stages (G, xa) of the column's slices once per task (warp prefix scan),
// and every row costs ONE table evaluation: lane l owns row 32 k + l of the
// band, evaluates Fn at the row's upper boundary and takes the lower one from
// lane l - 1 with a shuffle.  y(r, c) += (B ts(c)) (Fn_up - Fn_lo).
//
// Tiles and their overhang.  A footprint of at most three detector columns
// is processed ONCE, by the tile holding its first column: the tile's four
// own columns accumulate in registers, the two columns past the tile (its
// overhang) in shared memory, and the overhang is merged into the next
// tile's outputs by launch order (even tiles, then odd tiles: no atomics,
// no scratch; see the stores).  Wider footprints are taken by every tile
// they touch, own columns only.  Without the overhang a footprint was staged
// and evaluated by ~1.32 tiles on C3.
//
// Task decomposition, wedge enumeration and candidate setup follow round 1:
// one WARP owns (view, F3_CW-column tile, KR * 32-row band); it enumerates
// the wedge of voxel columns between the tile's edge rays, sets the
// candidates up lane-parallel (transverse weights in fp32, axial map in f64 at
// the (sub-)voxel centre, relative to the band), and gathers them into its
// register tile.  The next entry's x column is prefetched with cp.async while
// the current one is processed.  No atomics, no CTA barriers.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "sf_common.cuh"
#include "sf_launch.h"

#ifndef CTP_F3_MINB
#define CTP_F3_MINB 3
#endif

namespace ctp {

#ifndef CTP_F3_CW
#define CTP_F3_CW 4
#endif
constexpr int F3_CW = CTP_F3_CW;      // detector columns per tile (2 or 4)
static_assert(F3_CW == 2 || F3_CW == 4, "tile width");
// 32-row groups per warp task (KR, a template parameter): 24 (768-row bands)
// when every column's staged slices fit one piece (nz <= F3_XCAP), else 12
#ifndef CTP_F3_VCH
#define CTP_F3_VCH 16
#endif
#ifndef CTP_F3_PEND
#define CTP_F3_PEND 8  // (measured on C3: 16: 233.9 ms, 8: 231.6, 4: 231.6, 1: 232.0)
#endif
constexpr int F3_VCH = CTP_F3_VCH;    // views per chunk of the task order
constexpr int F3_PEND = CTP_F3_PEND;  // entries gathered before they are processed
#ifndef CTP_F3_WARPS
#define CTP_F3_WARPS 4
#endif
constexpr int F3_WARPS = CTP_F3_WARPS;  // independent warps per CTA (no CTA barriers: any count)
constexpr int F3_XCAP = 512;          // slices staged per piece (two 256-slice chunks)
#ifndef CTP_F3_BLK
#define CTP_F3_BLK 2
#endif
#ifndef CTP_F3_PAD
#define CTP_F3_PAD 160  // (a multiple of 4: 16-byte table stores)
#endif
constexpr int F3_BLK = CTP_F3_BLK;    // pairs of row groups per straight-line block (64 rows each)
constexpr int F3_PAD = CTP_F3_PAD;    // zero slices below / total slices above the staged range
static_assert(F3_PAD % 4 == 0, "16-byte aligned table stores");
constexpr int F3_TAB = F3_PAD + F3_XCAP + 4 + F3_PAD;  // G table length
constexpr int F3_OV = 2;                               // overhang columns (the next tile's first two)
constexpr int F3_EBUF = F3_PEND + 64;  // >= F3_PEND - 1 pending + 64 from one setup round


struct F3Entry {  // one (sub-)voxel column reaching the task's tile and band
  int col;        // x offset of the first staged slice za4 (float4 units on the vector path)
  int info;       // g0 | g1 << 5 | fast << 10 | inside << 11 | nst << 12 (nst staged slices; 0: misses the band)
  float cu;       // u(r + 1/2) = r invB + cu: upper boundary of band row r in staged-slice units
  float invB;     // 1 / rows per slice
  int resv;
  float a0, a1;   // amp(s) = lxy sqrt(1 + (a0 + a1 s)^2), s = staged slice index (lxy is in bts)
  unsigned gadj;   // the warp's G table base + F3_PAD - (bits of 1.5 * 2^23) entries (opaque; see f3_eval)
  float bts[F3_CW + F3_OV];  // B lxy ts(c) of columns c0 .. c0 + F3_CW + 1 (own + overhang 2; 0 outside)
  int has_ov;      // the overhang weights are not all zero
  int pad[5 - F3_CW];
};
static_assert(sizeof(F3Entry) == 64, "F3Entry layout");

struct F3Smem {  // per warp
  F3Entry ent[F3_EBUF];
  // staged slice j at index F3_PAD + j; [0, F3_PAD): 0 (written once),
  // [F3_PAD + n, F3_PAD + n + F3_PAD + 1]: the total (per entry).
  // Fn(u) = lerp(G_k, G_k+1, u - k).
  float G[F3_TAB];           // exclusive prefix of amp * x over the staged slices
  float xr[F3_XCAP];         // raw x of the next fast entry (cp.async; read by the staging, then refilled)
};
// after the per-warp F3Smem blocks, for the overhang kernels only: per warp
// float2 ov[32 KR] (rows x the next tile's first two columns)

__device__ __forceinline__ float2 sub2f_(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "sub.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}

// Candidate entry for this task: transverse weights of the tile's columns
// (fp32, sf_common.cuh) and the band-relative axial map in f64 at the
// (sub-)voxel centre.  Returns false if the (sub-)voxel misses the tile or
// the band.
__device__ __forceinline__ bool f3_fill(F3Entry& e, const SubFoot& f, const GridParams& gp, int col, int c0, int cw,
                                        const ViewAx& ax, float2 cxy, int rw0, int nrows, int band_rows, bool vec,
                                        bool ovmode, int ng) {
  // ovmode: a footprint of at most three columns belongs to the tile of its
  // first column (the columns past the tile are its overhang, merged into the
  // next tile's outputs); a wider one is taken by every tile it touches, own
  // columns only (and every footprint is, without ovmode)
  const bool narrow = ovmode && f.ch - f.cl <= F3_OV;
  if (narrow ? (f.cl < c0 || f.cl >= c0 + cw) : (max(f.cl, c0) > min(f.ch, c0 + cw - 1))) return false;
  double A, B;
  axial64(ax, gp.kind, (double)cxy.x, (double)cxy.y, A, B);
  A -= (double)rw0;  // row coordinate of slice 0's centre, band-relative
  // rows the column reaches (row r spans [r - .5, r + .5))
  const double top = A + B * ((double)gp.nz - 0.5);
  const double bot = A - 0.5 * B;
  const double rl = floor(bot + 0.5), rh = floor(top + 0.5);
  if (rh < 0.0 || rl > (double)(nrows - 1)) return false;
  const int r_lo = rl < 0.0 ? 0 : (int)rl, r_hi = rh > (double)(nrows - 1) ? nrows - 1 : (int)rh;
  // slices reaching band rows [0, nrows): one slice of slack on each side
  const double invB = 1.0 / B;
  int za = (int)floor((-0.5 - A) * invB - 0.5);
  int zb = (int)ceil(((double)nrows - 0.5 - A) * invB + 0.5);
  za = max(za, 0);
  zb = min(zb, gp.nz - 1);
  if (za > zb) return false;
  const int za4 = vec ? (za & ~3) : za;
  // (vector path: whole float4s -- nz and za4 are multiples of 4, so this
  // stays inside the column; the slices past zb reach no band row, see zb)
  const int nst = vec ? ((zb - za4 + 4) & ~3) : zb - za4 + 1;
  const double Lo = A + B * ((double)za4 - 0.5);  // lower boundary of staged slice 0
  e.cu = (float)((0.5 - Lo) * invB);
  e.invB = (float)invB;
  e.resv = 0;
  e.a1 = f.a1;
  e.a0 = fma_(f.a1, (float)za4, f.a0);
  e.gadj = 0u;
  const Trap p = make_trap(f);
  float ts[F3_CW + F3_OV];
  col_weights<F3_CW + F3_OV>(p, c0, ts);
  const float Bf = (float)B * f.lxy;  // the amplitude's constant factor, out of the staging
  bool ov = false;
#pragma unroll
  for (int c = 0; c < F3_CW + F3_OV; ++c) {
    const int cc = c0 + c;
    const bool mine = c < cw ? true : (narrow && cc < gp.nc);
    const bool on = mine && cc >= f.cl && cc <= f.ch;
    e.bts[c] = on ? Bf * ts[c] : 0.0f;
    if (c >= F3_CW && on) ov = true;
  }
  e.has_ov = ov ? 1 : 0;
  // x offset of slice za4 (32-bit: the launcher checks nx*ny*nz < 2^34 resp. 2^32)
  const unsigned xo = (unsigned)(((unsigned long long)(unsigned)col * (unsigned)gp.nz + (unsigned)za4) >> (vec ? 2 : 0));
  e.col = (int)xo;
  const int g0 = r_lo >> 5, g1 = r_hi >> 5;
  const bool fast = nst <= F3_XCAP;
  // inside: every row the gather evaluates (whole blocks of F3_BLK pairs
  // around [g0, g1]) maps into the padded table, so no clamps (f3_rows)
  const int q0 = (g0 >> 1) / F3_BLK, q1 = (g1 >> 1) / F3_BLK;
  const int rlo = 64 * F3_BLK * q0, rhi = min(64 * F3_BLK * (q1 + 1), band_rows) - 1;
  // (the vector path's table holds the total up to 128 ng + F3_PAD + 3)
  const bool inside = fmaf((float)rlo - 1.0f, e.invB, e.cu) >= 1.0f - (float)F3_PAD &&
                      fmaf((float)rhi, e.invB, e.cu) <= (float)((vec ? 128 * ng : nst) + F3_PAD) - 1.0f;
  e.info = g0 | (g1 << 5) | (fast ? (1 << 10) : 0) | (inside ? (1 << 11) : 0) | (nst << 12);
  return true;
}

// Lane-parallel setup of wedge candidates k = cbase + lane: owner primary
// index by binary search over the exclusive scan, footprint of the voxel
// column, compaction of the (sub-)footprints that reach the tile and band.
// Returns how many entries the warp added.  Out of line (its registers stay
// out of the gather loop).
__device__ __noinline__ int f3_candidates(const GridParams& gp, const ViewCoef* __restrict__ vcp,
                                          const ViewAx* __restrict__ vaxp, F3Entry* ent, int k, int total, int ib,
                                          int excl, int jl, bool primary_x, int c0, int cw, int rw0, int nrows,
                                          int band_rows, bool vec, bool ovmode, int ng, unsigned gadj) {
  const int lane = threadIdx.x & 31;
  int o = 0;
#pragma unroll
  for (int step = 16; step >= 1; step >>= 1) {
    const int ex = __shfl_sync(0xffffffffu, excl, o + step);
    if (ex <= k) o += step;
  }
  const int jo = __shfl_sync(0xffffffffu, jl, o);
  const int exo = __shfl_sync(0xffffffffu, excl, o);
  F3Entry e0, e1;
  int mask = 0;
  if (k < total) {
    const ViewCoef vc = *vcp;
    const ViewAx ax = *vaxp;
    const int ii = ib + o, j = jo + (k - exo);
    const int ix = primary_x ? ii : j, iy = primary_x ? j : ii;
    const int col = iy * gp.nx + ix;
    SubFoot f0, f1;
    float2 cxy0, cxy1;
    const int m = column_subs(vc, gp, ix, iy, f0, f1, cxy0, cxy1) & 3;
    if ((m & 1) && f3_fill(e0, f0, gp, col, c0, cw, ax, cxy0, rw0, nrows, band_rows, vec, ovmode, ng)) mask |= 1;
    if ((m & 2) && f3_fill(e1, f1, gp, col, c0, cw, ax, cxy1, rw0, nrows, band_rows, vec, ovmode, ng)) mask |= 2;
  }
  const int n = __popc(mask);
  const int ni = warp_incl_scan(n, lane);
  const int off = ni - n;
  e0.gadj = e1.gadj = gadj;
  if (mask & 1) ent[off] = e0;
  if (mask & 2) ent[off + (mask & 1)] = e1;
  return __shfl_sync(0xffffffffu, ni, 31);
}

// Stage (G, X) of n <= F3_XCAP slices: lane t takes slices 256 c + 4 t .. + 3
// and 256 c + 128 + 4 t .. + 3 of chunk c (512 contiguous bytes per 16-byte
// access), amp * x, local prefixes and two warp scans per chunk; G[n] ends up
// as the exclusive prefix at n (the total).
//   RAW (x in the cp.async buffer xraw, finite everywhere): slices >= n are
//   staged like the others -- they only change G / X past index n, which no
//   evaluation reads (u <= n, and at u = n the weight of X[n] is exactly 0).
//   Otherwise (global x): slices >= n read as 0 and X[n] = 0.
template <bool RAW, bool VEC>
__device__ __forceinline__ void f3_stage(F3Smem& S, const float* xraw, const float* __restrict__ xg, int n, float a0,
                                         float a1, int lane) {
  float carry = 0.0f;
#pragma unroll
  for (int c = 0; c < F3_XCAP / 256; ++c) {
    if (256 * c >= n) break;  // warp-uniform
    float2 xa[4];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int s = 256 * c + 128 * h + 4 * lane;
      float4 v = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      if (RAW) {
        v = *reinterpret_cast<const float4*>(xraw + s);
      } else if (s < n) {
        if (VEC) {
          v = __ldg(reinterpret_cast<const float4*>(xg + s));
        } else {
          v.x = __ldg(xg + s);
          if (s + 1 < n) v.y = __ldg(xg + s + 1);
          if (s + 2 < n) v.z = __ldg(xg + s + 2);
          if (s + 3 < n) v.w = __ldg(xg + s + 3);
        }
        if (s + 3 >= n) {  // slices past the staged range add nothing
          if (s + 1 >= n) v.y = 0.0f;
          if (s + 2 >= n) v.z = 0.0f;
          v.w = 0.0f;
        }
      }
      const float sf = (float)s;
      const float2 iA = make_float2(sf, sf + 1.0f), iB = make_float2(sf + 2.0f, sf + 3.0f);
      const float2 qA = fma2_(bc2_(a1), iA, bc2_(a0)), qB = fma2_(bc2_(a1), iB, bc2_(a0));
      const float2 tA = fma2_(qA, qA, bc2_(1.0f)), tB = fma2_(qB, qB, bc2_(1.0f));
      const float2 ampA = make_float2(sqrt_approx(tA.x), sqrt_approx(tA.y));
      const float2 ampB = make_float2(sqrt_approx(tB.x), sqrt_approx(tB.y));
      xa[2 * h] = mul2_(ampA, make_float2(v.x, v.y));
      xa[2 * h + 1] = mul2_(ampB, make_float2(v.z, v.w));
    }
    const float a_1 = xa[0].x, a_2 = a_1 + xa[0].y, a_3 = a_2 + xa[1].x, ta = a_3 + xa[1].y;
    const float b_1 = xa[2].x, b_2 = b_1 + xa[2].y, b_3 = b_2 + xa[3].x, tb = b_3 + xa[3].y;
    float ia = ta, ib = tb;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const float na = __shfl_up_sync(0xffffffffu, ia, d);
      const float nb = __shfl_up_sync(0xffffffffu, ib, d);
      if (lane >= d) {
        ia += na;
        ib += nb;
      }
    }
    const float tot_a = __shfl_sync(0xffffffffu, ia, 31);
    const float tot_b = __shfl_sync(0xffffffffu, ib, 31);
    const float ea = carry + (ia - ta), eb = (carry + tot_a) + (ib - tb);
    const float2 e01 = add2_(bc2_(ea), make_float2(0.0f, a_1)), e23 = add2_(bc2_(ea), make_float2(a_2, a_3));
    const float2 f01 = add2_(bc2_(eb), make_float2(0.0f, b_1)), f23 = add2_(bc2_(eb), make_float2(b_2, b_3));
    const int s0 = 256 * c + 4 * lane, s1 = s0 + 128;
    // RAW: the float4 that holds (or starts at) index n carries G[n]
    if (RAW ? s0 <= n : s0 < n)
      *reinterpret_cast<float4*>(S.G + F3_PAD + s0) = make_float4(e01.x, e01.y, e23.x, e23.y);
    if (RAW ? s1 <= n : s1 < n)
      *reinterpret_cast<float4*>(S.G + F3_PAD + s1) = make_float4(f01.x, f01.y, f23.x, f23.y);
    carry += tot_a + tot_b;
  }
  // back pad: entries n .. n + F3_PAD evaluate to the total (X = 0).  RAW:
  // the exclusive prefix at n is G[n] as stored above, unless no store
  // covered index n (n a multiple of 256), when it is the carry.
  __syncwarp();
  const float total = (!RAW || (n & 255) == 0) ? carry : S.G[F3_PAD + n];
  __syncwarp();
  for (int i = lane; i <= F3_PAD + 1; i += 32) S.G[F3_PAD + n + i] = total;  // (G_n+1 too: lerp)
}

// Inclusive warp scans of four series at once, step d: the predicated adds
// update the sums in place (no select / copy per series).
__device__ __forceinline__ void f3_scan_step4(float (&v)[4], int d) {
  asm("{.reg .pred p;\n\t.reg .f32 t0, t1, t2, t3;\n\t"
      "shfl.sync.up.b32 t0|p, %0, %4, 0, -1;\n\t"
      "shfl.sync.up.b32 t1, %1, %4, 0, -1;\n\t"
      "shfl.sync.up.b32 t2, %2, %4, 0, -1;\n\t"
      "shfl.sync.up.b32 t3, %3, %4, 0, -1;\n\t"
      "@p add.f32 %0, %0, t0;\n\t@p add.f32 %1, %1, t1;\n\t"
      "@p add.f32 %2, %2, t2;\n\t@p add.f32 %3, %3, t3;}"
      : "+f"(v[0]), "+f"(v[1]), "+f"(v[2]), "+f"(v[3]) : "r"(d));
}

// RAW staging of 128 NG slices (NG groups: the fewest that hold the entry's
// staged slices; short columns stage one or two groups) from the cp.async buffer, whose slices past
// the column's n are zero-filled by the copy (so G[k] = G[n], the total, for
// n <= k <= F3_XCAP without a fix-up), with the four 128-slice groups in
// flight: lane t owns slices 128 q + 4 t .. + 3 of group q; amp * x, local
// prefixes, four warp scans (only the final offsets chain).  The back pad
// past F3_XCAP holds the total.  Same values as f3_stage<true, *> for k <= n.
template <int NG>
__device__ __forceinline__ void f3_stage_raw(F3Smem& S, const float* xraw, float a0, float a1, float lanef4,
                                             int lane) {
  static_assert(F3_XCAP == 512 && (NG == 1 || NG == 2 || NG == 4), "one, two or four groups of 128 slices");
  static_assert((F3_PAD + 4) % 4 == 0 && (F3_PAD + 4) / 4 <= 64, "back pad: two float4 rounds");
  float p1[4], p2[4], p3[4], t[4], inc[4];
  // the slope factor q(s) = a0 + a1 s from the lane's first slice (no
  // per-slice index conversions)
  const float qb = fmaf(a1, lanef4, a0);
#pragma unroll
  for (int q = 0; q < NG; ++q) {
    const int s = 128 * q + 4 * lane;
    const float4 v = *reinterpret_cast<const float4*>(xraw + s);
    const float2 qA = make_float2(fmaf(a1, (float)(128 * q), qb), fmaf(a1, (float)(128 * q + 1), qb));
    const float2 qB = make_float2(fmaf(a1, (float)(128 * q + 2), qb), fmaf(a1, (float)(128 * q + 3), qb));
    const float2 tA = fma2_(qA, qA, bc2_(1.0f)), tB = fma2_(qB, qB, bc2_(1.0f));
    const float2 xa0 = mul2_(make_float2(sqrt_approx(tA.x), sqrt_approx(tA.y)), make_float2(v.x, v.y));
    const float2 xa1 = mul2_(make_float2(sqrt_approx(tB.x), sqrt_approx(tB.y)), make_float2(v.z, v.w));
    p1[q] = xa0.x;
    p2[q] = p1[q] + xa0.y;
    p3[q] = p2[q] + xa1.x;
    t[q] = p3[q] + xa1.y;
    inc[q] = t[q];
  }
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    if (NG == 4) {
      f3_scan_step4(inc, d);
    } else {
#pragma unroll
      for (int q = 0; q < NG; ++q) {
        const float nb = __shfl_up_sync(0xffffffffu, inc[q], d);
        if (lane >= d) inc[q] += nb;
      }
    }
  }
  float tot[4];
#pragma unroll
  for (int q = 0; q < NG; ++q) tot[q] = __shfl_sync(0xffffffffu, inc[q], 31);
  float base = 0.0f;
#pragma unroll
  for (int q = 0; q < NG; ++q) {
    const float e = base + (inc[q] - t[q]);
    const int s = 128 * q + 4 * lane;
    *reinterpret_cast<float4*>(S.G + F3_PAD + s) = make_float4(e, e + p1[q], e + p2[q], e + p3[q]);
    base += tot[q];
  }
  // back pad: entries 128 NG .. 128 NG + F3_PAD + 3 = the total
  float4* bp = reinterpret_cast<float4*>(S.G + F3_PAD + 128 * NG);
  const float4 tt = make_float4(base, base, base, base);
  bp[lane] = tt;
  if (lane < (F3_PAD + 4) / 4 - 32) bp[32 + lane] = tt;
}

// Fn(u) = G_k + (u - k) X_k, k = floor(u), -2^22 < u < 2^22: floor by adding
// 1.5 * 2^23 with round-down (the sum lies in [2^23, 2^24), where the float
// spacing is 1) and the signed index from the sum's bits (no conversion pipe).
// The table offset F3_PAD lives in g_adj (an integer), not in u, so u keeps
// its full fp32 resolution.
__device__ __forceinline__ float f3_eval(unsigned g_adj, float u) {
  const float tf = __fadd_rd(u, 12582912.0f);
  const float fr = u - (tf - 12582912.0f);  // both subtractions exact
  const unsigned a = (unsigned)__float_as_int(tf) * 4u + g_adj;
  float G0, G1;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(G0) : "r"(a));
  asm volatile("ld.shared.f32 %0, [%1 + 4];" : "=f"(G1) : "r"(a));
  return fmaf(fr, G1 - G0, G0);
}

// Rows 32 k + lane of the groups g0..g1, in blocks of four groups (a block
// outside [g0, g1] is skipped; inside one, every group is evaluated, rows
// beyond the column's reach clamp u to [0, n] and add exactly 0) and packed
// pairs of groups: acc(r, c) += bts(c) (Fn(u(r + .5)) - Fn(u(r - .5))).
__device__ __forceinline__ float2 f3_eval2(unsigned g_adj, float2 u) {
  float2 tf;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %4};\n\t"
      "add.rm.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(tf.x), "=f"(tf.y) : "f"(u.x), "f"(u.y), "f"(12582912.0f));
  const float2 fr = sub2f_(u, add2_(tf, bc2_(-12582912.0f)));  // exact
  const unsigned a0 = (unsigned)__float_as_int(tf.x) * 4u + g_adj;
  const unsigned a1 = (unsigned)__float_as_int(tf.y) * 4u + g_adj;
  float G0, H0, G1, H1;  // (G_k, G_k+1) of both boundaries
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(G0) : "r"(a0));
  asm volatile("ld.shared.f32 %0, [%1 + 4];" : "=f"(H0) : "r"(a0));
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(G1) : "r"(a1));
  asm volatile("ld.shared.f32 %0, [%1 + 4];" : "=f"(H1) : "r"(a1));
  const float2 G = make_float2(G0, G1);
  return fma2_(fr, sub2f_(make_float2(H0, H1), G), G);
}

// Rows of the groups g0..g1 in blocks of F3_BLK pairs of groups (64 rows each,
// straight-line code so the pairs' dependency chains interleave; blocks
// outside [g0, g1] are skipped).  In a pair (64 rows) lane l owns rows
// 64 p + 2 l and 64 p + 2 l + 1, evaluates Fn at their upper boundaries and
// takes the lower boundary of row 64 p + 2 l from lane l - 1 (lane 31 of the
// previous pair for lane 0).  Index k = floor(u) reads table entry F3_PAD + k;
// when every row of the evaluated blocks maps inside the
// pads (rows past the column's reach read the pads and add exactly 0),
// otherwise (CLAMP) u is clamped to [0, n].
template <int KR, bool CLAMP, bool OV>
__device__ __forceinline__ void f3_rows(float (&acc)[KR][F3_CW], float2* __restrict__ ovacc, unsigned g_adj,
                                        float cu, float invB, const float (&bts)[F3_CW + F3_OV], int n, int g0,
                                        int g1, int lane) {
  const float cuP = cu;
  const float ulo = 0.0f, uhi = (float)n;
  const float ua0 = fmaf((float)(2 * lane), invB, cuP), ub0 = fmaf((float)(2 * lane + 1), invB, cuP);
  const float du = 64.0f * invB;
  const int p0 = (g0 >> 1) / F3_BLK * F3_BLK, p1 = g1 >> 1;  // (p0: first pair of its block)
  // lower boundary of the first evaluated pair's first row (used by lane 0)
  float ul = fmaf(du, (float)p0, cuP - invB);
  if (CLAMP) ul = fminf(fmaxf(ul, ulo), uhi);
  float rot_prev = f3_eval(g_adj, ul);
  const int src = (lane + 31) & 31;
  const bool l0 = lane == 0;
  const float2 b01 = make_float2(bts[0], bts[1]);
  const float2 b23 = F3_CW == 4 ? make_float2(bts[2], bts[3]) : make_float2(0.0f, 0.0f);
  const float2 b45 = make_float2(bts[F3_CW], bts[F3_CW + 1]);  // overhang columns
  float4* ov4 = reinterpret_cast<float4*>(ovacc) + lane;  // rows 64 p + 2 lane, + 1 (two float2)
  constexpr int NB = (KR / 2 + F3_BLK - 1) / F3_BLK;
#pragma unroll
  for (int q = 0; q < NB; ++q) {  // blocks of F3_BLK pairs, straight-line inside
    if (F3_BLK * q + F3_BLK - 1 < p0 || F3_BLK * q > p1) continue;  // warp-uniform
#pragma unroll
    for (int p = F3_BLK * q; p < F3_BLK * q + F3_BLK && p < KR / 2; ++p) {
      float2 u = make_float2(fmaf(du, (float)p, ua0), fmaf(du, (float)p, ub0));
      if (CLAMP) {
        u.x = fminf(fmaxf(u.x, ulo), uhi);
        u.y = fminf(fmaxf(u.y, ulo), uhi);
      }
      const float2 F = f3_eval2(g_adj, u);
      const float rot = __shfl_sync(0xffffffffu, F.y, src);
      const float2 d = sub2f_(F, make_float2(l0 ? rot_prev : rot, F.x));
      rot_prev = rot;
      float2 a;
      a = fma2_(b01, bc2_(d.x), make_float2(acc[2 * p][0], acc[2 * p][1]));
      acc[2 * p][0] = a.x; acc[2 * p][1] = a.y;
      if (F3_CW == 4) {
        a = fma2_(b23, bc2_(d.x), make_float2(acc[2 * p][F3_CW - 2], acc[2 * p][F3_CW - 1]));
        acc[2 * p][F3_CW - 2] = a.x; acc[2 * p][F3_CW - 1] = a.y;
      }
      a = fma2_(b01, bc2_(d.y), make_float2(acc[2 * p + 1][0], acc[2 * p + 1][1]));
      acc[2 * p + 1][0] = a.x; acc[2 * p + 1][1] = a.y;
      if (F3_CW == 4) {
        a = fma2_(b23, bc2_(d.y), make_float2(acc[2 * p + 1][F3_CW - 2], acc[2 * p + 1][F3_CW - 1]));
        acc[2 * p + 1][F3_CW - 2] = a.x; acc[2 * p + 1][F3_CW - 1] = a.y;
      }
      if (OV) {  // the next tile's first two columns, accumulated in shared memory
        float4 o = ov4[32 * p];
        const float2 oa = fma2_(b45, bc2_(d.x), make_float2(o.x, o.y));
        const float2 ob = fma2_(b45, bc2_(d.y), make_float2(o.z, o.w));
        ov4[32 * p] = make_float4(oa.x, oa.y, ob.x, ob.y);
      }
    }
  }
}

template <int KR, bool VEC, int NG>
__device__ __forceinline__ void f3_process(F3Smem& S, float2* ovw, int nent, float (&acc)[KR][F3_CW],
                                           const float* __restrict__ xb, int lane) {
  // x of the next fast entry is in flight (cp.async, 16-byte copies on the
  // vector path) while the current one is processed
  auto next_fast = [&](int e) {
    for (; e < nent; ++e) {
      const int info = S.ent[e].info;
      if (info & (1 << 10)) {
        if (VEC) {
          const float* xc = xb + ((size_t)(unsigned)S.ent[e].col << 2);
          const int nst = info >> 12;
          // the whole buffer: float4s past nst (a multiple of 4 here) are
          // zero-filled, see f3_stage_raw
          const float* xl = xc + 4 * lane;
#pragma unroll
          for (int t = 0; t < NG; ++t) {  // the groups the staging reads
            const bool in = 4 * lane + 128 * t < nst;
            cp_async16_zfill(&S.xr[4 * lane + 128 * t], xl + (in ? 128 * t : 0), in ? 16u : 0u);
          }
          cp_async_commit();
        }
        return e;
      }
    }
    return nent;
  };
  const float lanef4 = (float)(4 * lane);
  int e_pf = next_fast(0);
  for (int e = 0; e < nent; ++e) {
    const F3Entry& E = S.ent[e];
    const int info = E.info;
    const int nst = info >> 12;
    if (nst == 0) continue;
    const float cu = E.cu, invB = E.invB, a0 = E.a0, a1 = E.a1;
    const unsigned g_adj = E.gadj;
    const int g0 = info & 31, g1 = (info >> 5) & 31;
    float bts[F3_CW + F3_OV];
#pragma unroll
    for (int c = 0; c < F3_CW + F3_OV; ++c) bts[c] = E.bts[c];
    const bool ov = E.has_ov != 0;
    const float* xg = xb + ((size_t)(unsigned)E.col << (VEC ? 2 : 0));
    if (e == e_pf) {  // fast: one piece, x staged by cp.async (vector path)
      const float* xraw = nullptr;
      if (VEC) {
        cp_async_wait_all();  // this lane's copies; the warp barrier publishes the others'
        __syncwarp();
        xraw = S.xr;
      }
      if (VEC) f3_stage_raw<NG>(S, xraw, a0, a1, lanef4, lane);
      else f3_stage<false, false>(S, nullptr, xg, nst, a0, a1, lane);
      __syncwarp();
      e_pf = next_fast(e + 1);  // loads for the next entry overlap this one
      if (info & (1 << 11)) {  // unclamped (see f3_fill)
        if (ov) f3_rows<KR, false, true>(acc, ovw, g_adj, cu, invB, bts, nst, g0, g1, lane);
        else f3_rows<KR, false, false>(acc, ovw, g_adj, cu, invB, bts, nst, g0, g1, lane);
      } else {
        if (ov) f3_rows<KR, true, true>(acc, ovw, g_adj, cu, invB, bts, nst, g0, g1, lane);
        else f3_rows<KR, true, false>(acc, ovw, g_adj, cu, invB, bts, nst, g0, g1, lane);
      }
      __syncwarp();
      continue;
    }
    // generic: pieces of F3_XCAP slices; each piece's clamped differences add
    // up to the whole column's (the integral is additive over pieces)
    for (int p0 = 0; p0 < nst; p0 += F3_XCAP) {
      const int n = min(F3_XCAP, nst - p0);
      f3_stage<false, false>(S, nullptr, xb + ((size_t)(unsigned)E.col << (VEC ? 2 : 0)) + p0, n,
                      fma_(a1, (float)p0, a0), a1, lane);
      __syncwarp();
      if (ov) f3_rows<KR, true, true>(acc, ovw, g_adj, cu - (float)p0, invB, bts, n, g0, g1, lane);
      else f3_rows<KR, true, false>(acc, ovw, g_adj, cu - (float)p0, invB, bts, n, g0, g1, lane);
      __syncwarp();
    }
  }
}

template <int KR, bool VEC, int NG>
__global__ void __launch_bounds__(F3_WARPS * 32, (KR * F3_CW > 48 ? 12 : 16) / F3_WARPS) sf_forward3d_kernel(
    const __grid_constant__ GridParams gp, const ViewCoef* __restrict__ vcoef, const ViewAx* __restrict__ vax,
    const float* __restrict__ xT, float* __restrict__ y, int accumulate, int parity, int tile_step,
    long long task0, long long ntasks) {
  extern __shared__ __align__(16) unsigned char f3_smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  F3Smem& S = reinterpret_cast<F3Smem*>(f3_smem_raw)[warp];
  const long long task = task0 + (long long)blockIdx.x * F3_WARPS + warp;
  if (task >= ntasks) return;  // warp-uniform; no CTA barriers in this kernel
  // this launch's tiles: every other one (parity 0: even, 1: odd; see the
  // stores at the end)
  // (tile_step 1: every tile, no overhang)
  const bool ovmode = tile_step == 2;
  const int ntiles = ((gp.nc + F3_CW - 1) / F3_CW + tile_step - 1 - parity) / tile_step;
  // band-major task order; within a band, chunks of F3_VCH consecutive views x
  // all tiles, so the CTAs resident at once cover a few degrees of rotation
  // whose wedges stay in L2
  const long long per_band = (long long)ntiles * gp.nv * gp.batch;
  const int band = (int)(task / per_band);
  const long long t2 = task % per_band;
  const int nvb = gp.nv * gp.batch;
  const int vch = (int)(t2 / ((long long)ntiles * F3_VCH));
  const int rem = (int)(t2 - (long long)vch * ntiles * F3_VCH);
  const int cv = min(F3_VCH, nvb - vch * F3_VCH);
  const int tile = rem / cv;
  const int vb = vch * F3_VCH + rem % cv;
  const int v = vb % gp.nv, b = vb / gp.nv;
  const int c0 = (tile_step * tile + parity) * F3_CW;
  const int cw = min(F3_CW, gp.nc - c0);
  const int rw0 = band * 32 * KR;
  const int nrows = min(32 * KR, gp.nr - rw0);
  const ViewCoef vc = vcoef[v];

  // wedge between the tile's edge rays, in (primary, secondary) grid axes
  float plx, ply, dlx, dly, phx, phy, dhx, dhy;
  edge_ray(vc, gp, (float)c0 - 0.5f, plx, ply, dlx, dly);
  edge_ray(vc, gp, (float)(c0 + cw) - 0.5f, phx, phy, dhx, dhy);
  const float nl = rsqrtf(dlx * dlx + dly * dly), nh = rsqrtf(dhx * dhx + dhy * dhy);
  const bool primary_x = fabsf(dlx) * nl + fabsf(dhx) * nh >= fabsf(dly) * nl + fabsf(dhy) * nh;
  const int nP = primary_x ? gp.nx : gp.ny, nQ = primary_x ? gp.ny : gp.nx;
  const float halfP = primary_x ? gp.half_x : gp.half_y, halfQ = primary_x ? gp.half_y : gp.half_x;
  const float lp = primary_x ? plx : ply, lq = primary_x ? ply : plx;
  const float ldp = primary_x ? dlx : dly, ldq = primary_x ? dly : dlx;
  const float hp = primary_x ? phx : phy, hq = primary_x ? phy : phx;
  const float hdp = primary_x ? dhx : dhy, hdq = primary_x ? dhy : dhx;
  const bool cull = vc.cull && fabsf(ldp) * nl > 1e-3f && fabsf(hdp) * nh > 1e-3f;
  const float lslope = cull ? ldq / ldp : 0.0f, hslope = cull ? hdq / hdp : 0.0f;

  static_assert(KR % 4 == 0 && KR <= 31, "blocks of two pairs of groups; 5-bit group indices in F3Entry::info");
  float acc[KR][F3_CW];
#pragma unroll
  for (int k = 0; k < KR; ++k)
#pragma unroll
    for (int c = 0; c < F3_CW; ++c) acc[k][c] = 0.0f;
  const float* xb = xT + (size_t)b * ((size_t)gp.nx * gp.ny) * gp.nz;
  // front pads of the G / X table (never rewritten); the RAW staging reads
  // the cp.async buffers past nst: keep them finite
  for (int i = lane; i < F3_PAD; i += 32) S.G[i] = 0.0f;
  float2* ovw = ovmode ? reinterpret_cast<float2*>(f3_smem_raw + sizeof(F3Smem) * F3_WARPS) + 32 * KR * warp
                      : nullptr;
  if (ovmode)
    for (int i = lane; i < 32 * KR; i += 32) ovw[i] = make_float2(0.0f, 0.0f);
  if (VEC)
    for (int i = lane; i < F3_XCAP; i += 32) S.xr[i] = 0.0f;
  __syncwarp();
  // G table base + F3_PAD entries - (bits of 1.5 * 2^23) entries; see f3_eval
  const unsigned g_adj = (unsigned)__cvta_generic_to_shared(S.G) + 4u * F3_PAD - 0x4B400000u * 4u;

  int pending = 0;
  for (int ib = 0; ib < nP; ib += 32) {
    // secondary-index range of primary index i on the two edge rays (+-1 margin)
    const int i = ib + lane;
    int jl = 0, cnt = 0;
    if (i < nP) {
      int jh = nQ - 1;
      if (cull) {
        const float pa = (float)i - halfP, pb = pa + 1.0f;
        const float q0 = lq + (pa - lp) * lslope, q1 = lq + (pb - lp) * lslope;
        const float q2 = hq + (pa - hp) * hslope, q3 = hq + (pb - hp) * hslope;
        const float qmin = fminf(fminf(q0, q1), fminf(q2, q3)) + halfQ;
        const float qmax = fmaxf(fmaxf(q0, q1), fmaxf(q2, q3)) + halfQ;
        if (qmin > -1e8f && qmax < 1e8f) {
          jl = max(jl, (int)floorf(qmin) - 1);
          jh = min(jh, (int)floorf(qmax) + 1);
        }
      }
      cnt = jh >= jl ? jh - jl + 1 : 0;
    }
    const int incl = warp_incl_scan(cnt, lane);
    const int excl = incl - cnt;
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    for (int cbase = 0; cbase < total; cbase += 32) {
      pending += f3_candidates(gp, vcoef + v, vax + v, S.ent + pending, cbase + lane, total, ib, excl, jl,
                               primary_x, c0, cw, rw0, nrows, 32 * KR, VEC, ovmode, NG, g_adj);
      __syncwarp();
      if (pending >= F3_PEND) {
        f3_process<KR, VEC, NG>(S, ovw, pending, acc, xb, lane);
        pending = 0;
        __syncwarp();
      }
    }
  }
  if (pending > 0) f3_process<KR, VEC, NG>(S, ovw, pending, acc, xb, lane);

  // store the tile: y[b][v][r][c0 + c], rows rw0 + 64 (k / 2) + 2 lane + k % 2.
  // Launch order makes the overhang merge deterministic without atomics:
  // parity 0 (even tiles) stores its own columns and its overhang into the
  // next (odd) tile's first two columns; parity 1 then adds its own first
  // two columns onto those, stores its last two, and adds its overhang onto
  // the next (even) tile's first two.  With `accumulate` every store adds.
  __syncwarp();
  float* yv = y + ((size_t)b * gp.nv + v) * (size_t)gp.nr * gp.nc;
  const bool v2 = (gp.nc & 1) == 0 && (reinterpret_cast<uintptr_t>(y) & 7) == 0;
  const bool ovc = ovmode && c0 + F3_CW < gp.nc;  // the next tile exists
#pragma unroll
  for (int k = 0; k < KR; ++k) {
    const int r = 64 * (k >> 1) + 2 * lane + (k & 1);
    if (r >= nrows) continue;
    float* row = yv + (size_t)(rw0 + r) * gp.nc + c0;
    const float2 o = ovc ? ovw[r] : make_float2(0.0f, 0.0f);
    if (v2 && cw == F3_CW) {
      float2 lo = make_float2(acc[k][0], acc[k][1]);
      if (accumulate || parity) lo = add2_(lo, *reinterpret_cast<const float2*>(row));
      *reinterpret_cast<float2*>(row) = lo;
      if (F3_CW == 4) {
        float2 hi = make_float2(acc[k][F3_CW - 2], acc[k][F3_CW - 1]);
        if (accumulate) hi = add2_(hi, *reinterpret_cast<const float2*>(row + 2));
        *reinterpret_cast<float2*>(row + 2) = hi;
      }
      if (ovc) {
        float2 n2 = o;
        if (accumulate || parity) n2 = add2_(n2, *reinterpret_cast<const float2*>(row + F3_CW));
        *reinterpret_cast<float2*>(row + F3_CW) = n2;
      }
    } else {
#pragma unroll
      for (int c = 0; c < F3_CW; ++c) {
        if (c >= cw) break;
        row[c] = (accumulate || (parity && c < F3_OV)) ? row[c] + acc[k][c] : acc[k][c];
      }
      if (ovc) {
        const int no = min(F3_OV, gp.nc - c0 - F3_CW);
        if (no > 0) row[F3_CW] = (accumulate || parity) ? row[F3_CW] + o.x : o.x;
        if (no > 1) row[F3_CW + 1] = (accumulate || parity) ? row[F3_CW + 1] + o.y : o.y;
      }
    }
  }
}

template <int KR>
static cudaError_t launch_forward3d(const GridParams& gp, const ViewCoef* vcoef, const ViewAx* vax, const float* xT,
                                   float* sino, int batch, bool accumulate, cudaStream_t st) {
  const size_t smem = sizeof(F3Smem) * F3_WARPS + sizeof(float2) * 32 * KR * F3_WARPS;
  // 16-byte x loads need every voxel column (nz floats) 16-byte aligned
  const bool vec = gp.nz % 4 == 0 && (reinterpret_cast<uintptr_t>(xT) & 15) == 0;
  if ((long long)gp.nx * gp.ny * gp.nz >= (vec ? (1LL << 34) : (1LL << 32))) return cudaErrorInvalidValue;
  if (gp.nz >= (1 << 19)) return cudaErrorInvalidValue;  // staged slice counts: 19 bits of F3Entry::info
  // 128-slice groups the vector path stages: the fewest that hold a column
  // (short columns stage one or two groups)
  auto kern = !vec ? sf_forward3d_kernel<KR, false, 4>
                   : (gp.nz <= 128 ? sf_forward3d_kernel<KR, true, 1>
                                   : (gp.nz <= 256 ? sf_forward3d_kernel<KR, true, 2> : sf_forward3d_kernel<KR, true, 4>));
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const long long nbands = (gp.nr + 32 * KR - 1) / (32 * KR);
  const long long ntiles_all = (gp.nc + F3_CW - 1) / F3_CW;
  const long long max_blocks = 1LL << 30;
  GridParams g2 = gp;
  g2.batch = batch;  // the task decode needs the batch extent
  // even tiles, then odd tiles (the overhang merge, see the kernel's stores)
  static const int step_env = getenv("CTP_F3_STEP") ? atoi(getenv("CTP_F3_STEP")) : 2;  // (A/B: 1 = no overhang)
  const int step = step_env == 1 ? 1 : 2;
  for (int parity = 0; parity < step; ++parity) {
    const long long ntiles = (ntiles_all + step - 1 - parity) / step;
    const long long ntasks = nbands * ntiles * (long long)gp.nv * batch;
    for (long long t0 = 0; t0 < ntasks; t0 += max_blocks * F3_WARPS) {
      const long long rem = ntasks - t0;
      const long long nb = (rem + F3_WARPS - 1) / F3_WARPS;
      const unsigned grid = (unsigned)(nb < max_blocks ? nb : max_blocks);
      kern<<<grid, F3_WARPS * 32, smem, st>>>(g2, vcoef, vax, xT, sino, accumulate ? 1 : 0, parity, step, t0,
                                              ntasks);
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_forward(const GridParams& gp, const ViewCoef* vcoef, const ViewAx* vax, const float* xT,
                           float* sino, int batch, bool accumulate, cudaStream_t st) {
  static const bool legacy = getenv("CTP_FWD_LEGACY") != nullptr;  // A/B against round 1's kernel
  if (legacy) return launch_forward_legacy(gp, vcoef, vax, xT, sino, batch, accumulate, st);
  // one 768-row band when every column fits one staged piece; else 384-row bands
  static const int kr_env = getenv("CTP_F3_KR") ? atoi(getenv("CTP_F3_KR")) : 0;  // (tuning)
  const bool wide = kr_env ? kr_env == 24 : (gp.nr > 384 && gp.nz <= F3_XCAP);
  return wide ? launch_forward3d<24>(gp, vcoef, vax, xT, sino, batch, accumulate, st)
              : launch_forward3d<12>(gp, vcoef, vax, xT, sino, batch, accumulate, st);
}

}  // namespace ctp
