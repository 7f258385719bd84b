// sf_kernels.cu -- sm_100a kernels of the SF-TR projector pair.
//
//   sf_back_kernel    : x = A^T y, voxel-driven GATHER (reference:
//                       sf_back_kernel, _kernels.py:666-763).  One warp owns one
//                       voxel column x BK_ZC slices (lanes along z) and loops
//                       over all views.  Footprint setup is LANE-PARALLEL: lane l
//                       sets up view vb+l, so one instruction stream prepares 32
//                       views; the per-view work is then a row-sum table
//                       Q(r) = sum_c ts(c) y[v][c][r] (coalesced, lanes along r)
//                       and K = rows_per_slice(B) fused multiply-adds per voxel.
//   sf_forward_kernel : y = A x, ray-driven GATHER (reference: per-view scatter
//                       into an f64 scratch, _kernels.py:555-663).  One CTA owns
//                       a detector tile (view, FW_CW columns, FW_ROWS rows),
//                       enumerates the voxel columns of the wedge that reaches
//                       the tile, sets them up one per thread, and each warp
//                       gathers its 32*FW_KR rows: P(r) = sum_iz tt(r,iz) amp x,
//                       y(r,c) += ts(c) P(r).
//   transpose_kernel  : [batch][R][C] -> [batch][C][R] layout change making the
//                       z (volume) / row (sinogram) axis contiguous.
//
// No atomics; every output element has one owner thread and a fixed
// summation order, so results are deterministic run to run.  Both kernels
// evaluate the coefficient (amp*tt)*ts from sf_common.cuh with identical
// operations, so the pair is an exact fp32 transpose.
#include <cuda_runtime.h>

#include <cstdint>

#include "sf_common.cuh"
#include "sf_launch.h"

#ifndef CTP_BK_MINB
#define CTP_BK_MINB 4  // resident CTAs/SM the back kernel is register-budgeted for
#endif
#ifndef CTP_FW_MINB
#define CTP_FW_MINB 4
#endif

namespace ctp {

// ---------------------------------------------------------------------------
// layout transpose
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) transpose_kernel(const float* __restrict__ in,
                                                        float* __restrict__ out, int R, int C,
                                                        int batch0, int rblock0) {
  __shared__ float tile[32][33];
  const int b = blockIdx.z + batch0;
  const size_t off = (size_t)b * (size_t)R * (size_t)C;
  const int c_base = blockIdx.x * 32, r_base = (blockIdx.y + rblock0) * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const int r = r_base + ty + k, c = c_base + tx;
    if (r < R && c < C) tile[ty + k][tx] = __ldg(in + off + (size_t)r * C + c);
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 32; k += 8) {
    const int c = c_base + ty + k, r = r_base + tx;
    if (r < R && c < C) out[off + (size_t)c * R + r] = tile[tx][ty + k];
  }
}

// ---------------------------------------------------------------------------
// back projection: x = A^T y
// ---------------------------------------------------------------------------
#ifndef CTP_BK_ZPL
#define CTP_BK_ZPL 8
#endif
#ifndef CTP_BK_WARPS
#define CTP_BK_WARPS 8
#endif
constexpr int BK_WARPS = CTP_BK_WARPS;  // warps per CTA (a 4 x BK_WARPS/4 block of voxel columns)
constexpr int BK_ZPL = CTP_BK_ZPL;      // voxels per lane
#ifndef CTP_BK_CX
#define CTP_BK_CX 1
#endif
constexpr int BK_CX = CTP_BK_CX;  // voxel columns along x per CTA (BK_WARPS / BK_CX along y)
static_assert(BK_WARPS % BK_CX == 0, "CTAs cover BK_CX x BK_WARPS/BK_CX voxel columns");
constexpr int BK_ZC = 32 * BK_ZPL;  // slices per warp
static_assert(BK_ZC == kBackZBlock, "sf_launch.h advertises the z-block size");
#ifndef CTP_BK_QMAX
#define CTP_BK_QMAX (BK_ZC * 25 / 16)  // rows covered by slices with B <= 1.5 (+ margin)
#endif
constexpr int BK_QMAX = CTP_BK_QMAX;  // per-warp row-sum table (rows) for the fast path
constexpr int BK_NCF = 4;           // footprint columns handled by the table path

struct BkEntry {  // one (sub-)voxel footprint of the warp's column in one view
  float A, B, E, lxy;
  float a0, a1;
  int cl;
  int ncol;  // 0: no contribution; > BK_NCF: wide footprint (direct path)
  float ts[BK_NCF];  // 0 beyond ncol
  // precomputed by the lane-parallel setup for the fast path:
  int off0;  // (cl * nr + ra4): element offset of the first table row, column cl
  int pk;    // bit 0: fast path; bits 1-3: K; bits 4-15: n4; bits 16-31: ra4
  int pad[2];
};
static_assert(sizeof(BkEntry) == 64, "BkEntry layout");

struct BkSmem {
  BkEntry ents[BK_WARPS][32];          // lane-parallel setup of 32 views, per warp
  BkEntry split[BK_WARPS];             // second sub-footprint of a split voxel (rare)
  float qbuf[BK_WARPS][BK_QMAX + 8];   // per-warp row-sum table Q(r)
};

// One entry of the lane-parallel setup.  With `ax` (3D back kernel) the
// axial map is taken in f64 at the (sub-)voxel centre and stored RELATIVE to
// a local origin: rows counted from `origin` (= the 4-aligned first table
// row, kept in pad[1]) and slices counted from izs, so that
// T = A + B * (iz - izs) stays below ~B * 32 * BK_ZPL rows in magnitude and
// fp32 resolves footprint edges to ~1e-5 row even on 1536-row detectors
// (round 1 used absolute row coordinates: 1.2e-4 row at C5).  Without `ax`
// (fan kernels: one slice, one row) the f32 absolute map is kept.
__device__ __forceinline__ void fill_entry(BkEntry& e, const SubFoot& f, const GridParams& gp, int izs, int ize,
                                           const ViewAx* ax = nullptr, float2 cxy = make_float2(0.0f, 0.0f)) {
  e.A = f.A; e.B = f.B; e.E = f.E; e.lxy = f.lxy; e.a0 = f.a0; e.a1 = f.a1;
  e.cl = f.cl;
  e.ncol = f.ch >= f.cl ? f.ch - f.cl + 1 : 0;
  const Trap p = make_trap(f);
  float ts[BK_NCF];
  col_weights<BK_NCF>(p, f.cl, ts);
#pragma unroll
  for (int k = 0; k < BK_NCF; ++k) e.ts[k] = k < e.ncol ? ts[k] : 0.0f;
  const int K = rows_per_slice(f.B);
  int Ra, Rz;
  if (ax) {
    double A, B;
    axial64(*ax, gp.kind, (double)cxy.x, (double)cxy.y, A, B);
    const double Ts = fma(B, (double)izs, A), Te = fma(B, (double)ize, A);
    Ra = (int)floor(Ts - 0.5 * B - 0.5) + 1;
    Rz = (int)floor(Te - 0.5 * B - 0.5) + 1 + K - 1;
    const int origin = Ra & ~3;
    e.A = (float)(Ts - (double)origin);
    e.B = (float)B;
    e.E = (float)(0.5 * B);
    e.a0 = fma_(f.a1, (float)izs, f.a0);
    e.pad[1] = origin;
  } else {
    Ra = first_row(sub_(fma_(f.B, (float)izs, f.A), f.E));
    Rz = first_row(sub_(fma_(f.B, (float)ize, f.A), f.E)) + K - 1;
    e.pad[1] = 0;
  }
  const int ra4 = Ra & ~3;
  const int n4 = ((Rz | 3) - ra4 + 1) >> 2;
  const bool fast = e.ncol > 0 && e.ncol <= BK_NCF && f.cl + 3 <= gp.nc - 1 && K <= 4 && Ra >= 0 &&
                    Rz < gp.nr && (gp.nr & 3) == 0 && 4 * n4 <= BK_QMAX + 8 && n4 < 4096;
  e.pk = fast ? (1 | (K << 1) | (n4 << 4) | (ra4 << 16)) : 0;
  e.off0 = fast ? f.cl * gp.nr + ra4 : 0;
  if (Rz < 0 || Ra > gp.nr - 1) e.ncol = 0;  // entirely off the detector
}

// Direct (table-free) contribution of one voxel: rows r0..r0+K-1, any
// footprint width.  Same operations, in the same order, as the table path.
__device__ __noinline__ float back_voxel_direct(float acc, float amp, float lo, float hi,
                                                const BkEntry& e, const Trap& wide, int K,
                                                const float* __restrict__ yv, int nr, int origin) {
  const float fl = row_floor(lo);  // r0 - 1 (rows relative to origin)
  const int r0 = (int)fl + 1 + origin;
  float g = clampf_(add_(fl, 0.5f), lo, hi);
  for (int k = 0; k < K; ++k) {
    const int r = r0 + k;
    const float gn = clampf_(add_(fl, (float)k + 1.5f), lo, hi);
    float q = 0.0f;
    if (r >= 0 && r < nr) {
      if (e.ncol <= BK_NCF) {
        for (int c = 0; c < e.ncol; ++c) q = fma_(e.ts[c], __ldg(yv + (size_t)(e.cl + c) * nr + r), q);
      } else {
        float prev = trap_cum(wide, sub_((float)e.cl, 0.5f));
        for (int c = 0; c < e.ncol; ++c) {
          const float cur = trap_cum(wide, add_((float)(e.cl + c), 0.5f));
          q = fma_(sub_(cur, prev), __ldg(yv + (size_t)(e.cl + c) * nr + r), q);
          prev = cur;
        }
      }
    }
    acc = fma_(mul_(amp, sub_(gn, g)), q, acc);
    g = gn;
  }
  return acc;
}

// Table path for a PAIR of slices (izf.x, izf.y), packed f32x2: each slice
// adds sum_k (amp * tt_k) * Q(r0 + k) over its K rows.  The boundaries of row
// r0 + k are fl + 0.5 + k and fl + 1.5 + k (fl = r0 - 1); the lowest one is
// <= lo and the highest >= hi by construction, so their clamps are exactly lo
// and hi, and every tt_k equals clamp(r+.5,lo,hi) - clamp(r-.5,lo,hi) as the
// forward kernel evaluates it.
template <int K>
__device__ __forceinline__ float2 back_pair_rows(float2 acc, const BkEntry& e, float2 izf,
                                                 const float* qw, int Ra) {
  const float2 T = fma2_(bc2_(e.B), izf, bc2_(e.A));
  const float2 lo = add2_(T, bc2_(-e.E)), hi = add2_(T, bc2_(e.E));
  const float2 q = fma2_(bc2_(e.a1), izf, bc2_(e.a0));
  const float2 t = fma2_(q, q, bc2_(1.0f));
  const float2 amp = mul2_(bc2_(e.lxy), make_float2(sqrt_approx(t.x), sqrt_approx(t.y)));
  const float2 lm = add2_(lo, bc2_(-0.5f));
  const float2 fl = make_float2(floorf(lm.x), floorf(lm.y));
  const float* qa = qw + ((int)fl.x + 1 - Ra);
  const float* qb = qw + ((int)fl.y + 1 - Ra);
  float2 g = lo;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    float2 gn;
    if (k == K - 1) {
      gn = hi;
    } else {
      const float2 bnd = add2_(fl, bc2_((float)k + 1.5f));
      // bnd = fl + k + 1.5 > lo always (fl = floor(lo - .5) > lo - 1.5), so
      // clamp(bnd, lo, hi) is exactly min(bnd, hi)
      gn = make_float2(fminf(bnd.x, hi.x), fminf(bnd.y, hi.y));
    }
    const float2 c = mul2_(amp, add2_(gn, make_float2(-g.x, -g.y)));
    acc = fma2_(c, make_float2(qa[k], qb[k]), acc);
    g = gn;
  }
  return acc;
}

// single slice (tail of an odd count), same operations
template <int K>
__device__ __forceinline__ float back_one_rows(float acc, const BkEntry& e, float izf,
                                               const float* qw, int Ra) {
  const float T = fma_(e.B, izf, e.A);
  const float lo = add_(T, -e.E), hi = add_(T, e.E);
  const float q = fma_(e.a1, izf, e.a0);
  const float amp = mul_(e.lxy, sqrt_approx(fma_(q, q, 1.0f)));
  const float fl = floorf(add_(lo, -0.5f));
  const float* qa = qw + ((int)fl + 1 - Ra);
  float g = lo;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const float gn = (k == K - 1) ? hi : fminf(add_(fl, (float)k + 1.5f), hi);  // (> lo, see above)
    acc = fma_(mul_(amp, add_(gn, -g)), qa[k], acc);
    g = gn;
  }
  return acc;
}

template <int K>
#ifndef CTP_BK_FULL
#define CTP_BK_FULL 1  // straight-line slice pairs when every lane has BK_ZPL slices
#endif
__device__ __forceinline__ void back_slices(float (&acc)[BK_ZPL], const BkEntry& e, float izf0,
                                            int nvalid, const float* qw, int Ra) {
#if CTP_BK_FULL
  if (__all_sync(0xffffffffu, nvalid == BK_ZPL)) {  // the pair chains interleave
#pragma unroll
    for (int m = 0; m < BK_ZPL; m += 2) {
      const float2 r = back_pair_rows<K>(make_float2(acc[m], acc[m + 1]), e,
                                         make_float2(izf0 + (float)(32 * m), izf0 + (float)(32 * m + 32)),
                                         qw, Ra);
      acc[m] = r.x;
      acc[m + 1] = r.y;
    }
    return;
  }
#endif
#pragma unroll
  for (int m = 0; m < BK_ZPL; m += 2) {
    if (m + 1 < nvalid) {
      const float2 r = back_pair_rows<K>(make_float2(acc[m], acc[m + 1]), e,
                                         make_float2(izf0 + (float)(32 * m), izf0 + (float)(32 * m + 32)),
                                         qw, Ra);
      acc[m] = r.x;
      acc[m + 1] = r.y;
    } else if (m < nvalid) {
      acc[m] = back_one_rows<K>(acc[m], e, izf0 + (float)(32 * m), qw, Ra);
    }
  }
}

// Q(r) for 4 consecutive rows per lane and iteration (16-byte loads) over the
// NC footprint columns: Q = ((t0 y0 + t1 y1) + ...) in fixed column order
template <int NC>
__device__ __forceinline__ void row_sums(float4* q4, const float* yv, int nr, const float (&ts)[BK_NCF],
                                         int n4, int lane) {
  const float4* v[NC];
  float2 T[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    v[k] = reinterpret_cast<const float4*>(yv + k * nr);
    T[k] = bc2_(ts[k]);
  }
#pragma unroll 1
  for (int t = lane; t < n4; t += 32) {
    float4 a[NC];
#pragma unroll
    for (int k = 0; k < NC; ++k) a[k] = __ldg(v[k] + t);
    float2 lo = mul2_(T[0], make_float2(a[0].x, a[0].y));
    float2 hi = mul2_(T[0], make_float2(a[0].z, a[0].w));
#pragma unroll
    for (int k = 1; k < NC; ++k) {
      lo = fma2_(T[k], make_float2(a[k].x, a[k].y), lo);
      hi = fma2_(T[k], make_float2(a[k].z, a[k].w), hi);
    }
    q4[t] = make_float4(lo.x, lo.y, hi.x, hi.y);
  }
}

// Lane-parallel footprint setup of one voxel column for views vb + lane: the
// entries of this lane's view go to e[0] (and e[1] for a split voxel).
// Returns whether any lane of the warp has a split voxel.  Out of line: it is
// run once per 32 views, and keeping its register-hungry geometry out of the
// per-view loop leaves that loop's registers alone.
__device__ __noinline__ bool back_setup(const GridParams& gp, const ViewCoef* __restrict__ vcoef, int vb,
                                        int ix, int iy, int izs, int ize, BkEntry* e) {
  const int v = vb + (threadIdx.x & 31);
  BkEntry e0, e1;
  e0.ncol = 0;
  e0.pk = 0;
  e1.ncol = 0;
  e1.pk = 0;
  int mask = 0;
  if (v < gp.nv) {
    const ViewCoef vc = vcoef[v];
    SubFoot f0, f1;
    mask = column_footprint(vc, gp, ix, iy, f0, f1);
    if (mask & 1) fill_entry(e0, f0, gp, izs, ize);
    if (mask & 2) fill_entry(e1, f1, gp, izs, ize);
  }
  e[0] = e0;
  const bool split = __any_sync(0xffffffffu, (mask & 2) != 0);
  if (split) e[1] = e1;
  return split;
}

// 3D back kernel variant of back_setup: only the first sub-footprint is kept
// (its mask in pad[0]); the second one of a split voxel is rebuilt in the
// view loop when needed, which halves the entry table (more L1 for y rows)
__device__ __noinline__ bool back_setup1(const GridParams& gp, const ViewCoef* __restrict__ vcoef,
                                         const ViewAx* __restrict__ vax, int vb, int ix, int iy, int izs, int ize,
                                         BkEntry* e) {
  const int v = vb + (threadIdx.x & 31);
  BkEntry e0;
  e0.ncol = 0;
  e0.pk = 0;
  e0.pad[1] = 0;
  int mask = 0;
  if (v < gp.nv) {
    const ViewCoef vc = vcoef[v];
    SubFoot f0, f1;
    float2 c0, c1;
    mask = column_subs(vc, gp, ix, iy, f0, f1, c0, c1) & 3;
    if (mask & 1) fill_entry(e0, f0, gp, izs, ize, vax + v, c0);
  }
  e0.pad[0] = mask;
  *e = e0;
  return __any_sync(0xffffffffu, (mask & 2) != 0);
}

__global__ void __launch_bounds__(BK_WARPS * 32, CTP_BK_MINB) sf_back_kernel(
    const __grid_constant__ GridParams gp, const ViewCoef* __restrict__ vcoef, const ViewAx* __restrict__ vax,
    const float* __restrict__ yT, float* __restrict__ out, int accumulate, int z0, int z1) {
  extern __shared__ __align__(16) unsigned char bk_smem_raw[];
  BkSmem& SM = *reinterpret_cast<BkSmem*>(bk_smem_raw);
  auto& ents = SM.ents;
  auto& qbuf = SM.qbuf;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nbx = (gp.nx + BK_CX - 1) / BK_CX;
  const int ix = (blockIdx.x % nbx) * BK_CX + (warp % BK_CX);
  const int iy = (blockIdx.x / nbx) * (BK_WARPS / BK_CX) + (warp / BK_CX);
  if (ix >= gp.nx || iy >= gp.ny) return;  // warp-uniform; no CTA barriers below
  const int b = blockIdx.z;
  const int izs = z0 + blockIdx.y * BK_ZC;  // slices [z0, z1) of this launch
  const int ize = min(izs + BK_ZC, z1) - 1;
  const int nr = gp.nr, nc = gp.nc;
  const size_t view_elems = (size_t)nc * nr;
  const float* yb = yT + (size_t)b * gp.nv * view_elems;
  float* qw = qbuf[warp];
  BkEntry(&my)[32] = ents[warp];
  BkEntry& sp = SM.split[warp];
  // this lane's slices: izs + lane + 32 m, m < nvalid; entries count slices
  // from izs and rows from a per-entry origin (fill_entry)
  const int span = ize - izs - lane;  // may be negative when nz < 32
  const int nvalid = span < 0 ? 0 : min(BK_ZPL, span / 32 + 1);
  const float izf0 = (float)lane;
  float acc[BK_ZPL];
#pragma unroll
  for (int m = 0; m < BK_ZPL; ++m) acc[m] = 0.0f;

  for (int vb = 0; vb < gp.nv; vb += 32) {
    // ---- lane-parallel footprint setup: lane l <- view vb + l
    // nsub = 2 when any view of this batch splits the voxel (_sf_subdivide), else 1
    const int nsub = back_setup1(gp, vcoef, vax, vb, ix, iy, izs, ize, &my[lane]) ? 2 : 1;
    __syncwarp();
    const int nvb = min(32, gp.nv - vb);
    const float* yview = yb + (size_t)vb * view_elems;  // [c][r] of view vb + j
    for (int j = 0; j < nvb; ++j, yview += view_elems) {
#pragma unroll 1
      for (int s = 0; s < nsub; ++s) {
        if (s == 1) {  // the second half of a split voxel (_sf_subdivide), rebuilt
          if (!(my[j].pad[0] & 2)) continue;
          __syncwarp();  // every lane is done with the previous split entry
          if (lane == 0) {
            SubFoot f0, f1;
            float2 c0, c1;
            column_subs(vcoef[vb + j], gp, ix, iy, f0, f1, c0, c1);
            fill_entry(sp, f1, gp, izs, ize, vax + vb + j, c1);
          }
          __syncwarp();
        }
        const BkEntry& ef = s == 0 ? my[j] : sp;
        const int pk = ef.pk;
        if (pk & 1) {
          // fast path: everything precomputed; 4-row float4 row sums, then slices
          const float* yv = yview + ef.off0;
          const int n4 = (pk >> 4) & 0xfff;
          float4* q4 = reinterpret_cast<float4*>(qw);
          switch (ef.ncol) {  // warp-uniform: load only the footprint's columns
            case 1: row_sums<1>(q4, yv, nr, ef.ts, n4, lane); break;
            case 2: row_sums<2>(q4, yv, nr, ef.ts, n4, lane); break;
            case 3: row_sums<3>(q4, yv, nr, ef.ts, n4, lane); break;
            default: row_sums<4>(q4, yv, nr, ef.ts, n4, lane); break;
          }
          __syncwarp();
          // the table starts at the entry's row origin (ra4): relative row 0
          const int K = (pk >> 1) & 7;
          const BkEntry e = ef;
          if (K == 2) back_slices<2>(acc, e, izf0, nvalid, qw, 0);
          else if (K == 3) back_slices<3>(acc, e, izf0, nvalid, qw, 0);
          else back_slices<4>(acc, e, izf0, nvalid, qw, 0);
          __syncwarp();
          continue;
        }
        if (ef.ncol == 0) continue;
        const BkEntry& e = ef;  // (shared memory: no private copy on the rare paths)
        const int K = rows_per_slice(e.B);
        const int origin = e.pad[1];
        const int Rar = first_row(sub_(e.A, e.E));  // relative to origin
        const int Ra = Rar + origin;
        const int Rz = first_row(sub_(fma_(e.B, (float)(ize - izs), e.A), e.E)) + K - 1 + origin;
        if (Rz < 0 || Ra > nr - 1) continue;
        const float* yv = yview;  // [c][r] of the view
        const int nq = Rz - Ra + 1;
        if (nq <= BK_QMAX && e.ncol <= BK_NCF && K <= 4) {
          // row sums Q(r) = sum_k ts_k y[cl+k][r]; absent columns have ts = 0 and
          // read a clamped (valid) column, adding exactly 0
          const float* p0 = yv + (size_t)e.cl * nr;
          const float* p1 = yv + (size_t)min(e.cl + 1, nc - 1) * nr;
          const float* p2 = yv + (size_t)min(e.cl + 2, nc - 1) * nr;
          const float* p3 = yv + (size_t)min(e.cl + 3, nc - 1) * nr;
          const float t0 = e.ts[0];
          const float t1 = e.ncol > 1 ? e.ts[1] : 0.0f;
          const float t2 = e.ncol > 2 ? e.ts[2] : 0.0f;
          const float t3 = e.ncol > 3 ? e.ts[3] : 0.0f;
          if (Ra >= 0 && Rz < nr) {
            // rows r and r + 32 per iteration, packed
            const float2 T0 = bc2_(t0), T1 = bc2_(t1), T2 = bc2_(t2), T3 = bc2_(t3);
#pragma unroll 2
            for (int t = lane; t < nq; t += 64) {
              const int r = Ra + t;
              const bool two = t + 32 < nq;
              const int r2 = two ? r + 32 : r;
              float2 q = mul2_(T0, make_float2(__ldg(p0 + r), __ldg(p0 + r2)));
              q = fma2_(T1, make_float2(__ldg(p1 + r), __ldg(p1 + r2)), q);
              q = fma2_(T2, make_float2(__ldg(p2 + r), __ldg(p2 + r2)), q);
              q = fma2_(T3, make_float2(__ldg(p3 + r), __ldg(p3 + r2)), q);
              qw[t] = q.x;
              if (two) qw[t + 32] = q.y;
            }
          } else {
#pragma unroll 4
            for (int t = lane; t < nq; t += 32) {
              const int r = Ra + t;
              const bool in = (unsigned)r < (unsigned)nr;
              const int rr = in ? r : 0;
              float q = mul_(t0, __ldg(p0 + rr));
              q = fma_(t1, __ldg(p1 + rr), q);
              q = fma_(t2, __ldg(p2 + rr), q);
              q = fma_(t3, __ldg(p3 + rr), q);
              qw[t] = in ? q : 0.0f;
            }
          }
          __syncwarp();
          if (K == 2) back_slices<2>(acc, e, izf0, nvalid, qw, Rar);
          else if (K == 3) back_slices<3>(acc, e, izf0, nvalid, qw, Rar);
          else back_slices<4>(acc, e, izf0, nvalid, qw, Rar);
          __syncwarp();
        } else {
          Trap wide{};
          if (e.ncol > BK_NCF) {  // rare: rebuild the breakpoints of this footprint
            SubFoot f0, f1;
            const int mask = column_footprint(vcoef[vb + j], gp, ix, iy, f0, f1);
            (void)mask;
            wide = make_trap(s == 0 ? f0 : f1);
          }
          for (int m = 0; m < BK_ZPL; ++m) {
            if (m >= nvalid) break;
            const float izf = izf0 + (float)(32 * m);
            const float T = fma_(e.B, izf, e.A);
            const float lo = sub_(T, e.E), hi = add_(T, e.E);
            const float q = fma_(e.a1, izf, e.a0);
            const float amp = mul_(e.lxy, sqrt_approx(fma_(q, q, 1.0f)));
            acc[m] = back_voxel_direct(acc[m], amp, lo, hi, e, wide, K, yv, nr, origin);
          }
        }
      }
    }
    __syncwarp();
  }
  // out[b][iz][iy][ix]
  const size_t plane = (size_t)gp.ny * gp.nx;
  float* ob = out + (size_t)b * plane * gp.nz + (size_t)iy * gp.nx + ix;
#pragma unroll
  for (int m = 0; m < BK_ZPL; ++m) {
    if (m >= nvalid) break;
    float* p = ob + (size_t)(izs + lane + 32 * m) * plane;
    *p = accumulate ? (*p + acc[m]) : acc[m];
  }
}

// ---------------------------------------------------------------------------
// forward projection: y = A x
// ---------------------------------------------------------------------------
#ifndef CTP_FW_CW
#define CTP_FW_CW 4
#endif
constexpr int FW_CW = CTP_FW_CW;  // detector columns per tile
#ifndef CTP_FW_KR
#define CTP_FW_KR 12
#endif
constexpr int FW_KR = CTP_FW_KR;     // 32-row groups per warp
constexpr int FW_ROWS = 32 * FW_KR;  // rows per warp task
#ifndef CTP_FW_VCH
#define CTP_FW_VCH 16  // views per chunk of the task order (0: view-major within a band)
#endif
constexpr int FW_VCH = CTP_FW_VCH;
static_assert(FW_KR <= 32, "row groups are 5-bit in FwEntry::info");
constexpr int FW_XPAD = 4;           // zero slots below the staged slices
// slices staged per entry (fast path) or per piece (generic path): the band's
// rows plus slack for B < 1, rounded to whole 128-slice vector loads
constexpr int FW_XCAP = ((32 * FW_KR + 64) + 127) / 128 * 128;
constexpr int FW_XLEN = FW_XPAD + FW_XCAP + 4;  // + zero slots above
constexpr int FW_NLD = FW_XCAP / 128;           // float4 x loads per lane (fast path)
#ifndef CTP_FW_SG
#define CTP_FW_SG 1  // staging loads per branch
#endif
constexpr int FW_SG = CTP_FW_SG;
static_assert(FW_NLD % FW_SG == 0, "staging loads are processed in groups of FW_SG");

struct FwEntry {
  int col;   // iy*nx + ix; band_info turns it into the x offset col*nz + za4 of the first staged slice
  int za4;   // first staged slice (a multiple of 4 on the vector path)
  int nst;   // staged slices: za4 .. za4 + nst - 1 (0: the entry misses the band)
  int info;  // g0 | g1 << 5 | ncand << 10 | fast << 17 (band-specific, see band_info)
  float A, B, E;
  float lxy, a0, a1;
  float invB, cb;   // candidate slices of row r start at floor(r*invB + cb) + 1
  float ts[FW_CW];  // weights of the tile's columns (0 outside the footprint)
};
static_assert(sizeof(FwEntry) == 48 + 4 * FW_CW, "FwEntry layout");

__device__ __forceinline__ bool reaches_tile(const SubFoot& f, const GridParams& gp, int c0, int cw,
                                             float band_lo, float band_hi) {
  const bool cols_ok = max(f.cl, c0) <= min(f.ch, c0 + cw - 1);
  const float tlo = sub_(row_center(f, 0), f.E);
  const float thi = add_(row_center(f, gp.nz - 1), f.E);
  return cols_ok && thi > band_lo && tlo < band_hi;
}

// Candidate slices per row.  Slice iz overlaps row r only if iz lies in the
// open interval ((r - .5 - E - A)/B, (r + .5 + E - A)/B) of length
// L = (1 + 2E)/B; the candidates floor(s - 0.01) + 1 ... + ceil(L + 0.02) cover
// it (an open interval of length L holds at most ceil(L) integers; the 0.01 /
// 0.02 margins absorb fp32 rounding of lo / hi and of the interval ends).
__device__ __forceinline__ int cand_count(float E, float invB) {
  return (int)ceilf((1.0f + 2.0f * E) * invB + 0.02f);
}

__device__ __forceinline__ void write_entry(FwEntry& e, const SubFoot& f, int col, int c0, int cw) {
  e.col = col;
  e.A = f.A; e.B = f.B; e.E = f.E;
  e.lxy = f.lxy; e.a0 = f.a0; e.a1 = f.a1;
  const float invB = 1.0f / f.B;
  e.invB = invB;
  e.cb = (-0.5f - f.E - f.A) * invB - 0.01f;
  const Trap p = make_trap(f);
  float ts[FW_CW];
  col_weights<FW_CW>(p, c0, ts);
  const int lo = max(f.cl, c0), hi = min(f.ch, c0 + cw - 1);
#pragma unroll
  for (int c = 0; c < FW_CW; ++c) {
    const int cc = c0 + c;
    e.ts[c] = (cc >= lo && cc <= hi) ? ts[c] : 0.0f;
  }
  e.za4 = 0;
  e.nst = 0;
  e.info = 0;
}

// 3D forward: replace the entry's f32 absolute axial map by the f64 one at
// the (sub-)voxel centre, RELATIVE to the band's first row rw0 (the kernel
// then counts rows from rw0), so fp32 resolves footprint edges to ~1e-5 row
// on 1536-row detectors (round 1: absolute rows, 1.2e-4 row at C5).
__device__ __forceinline__ void localize_entry(FwEntry& e, const ViewAx& ax, const GridParams& gp, float2 cxy,
                                               int rw0) {
  double A, B;
  axial64(ax, gp.kind, (double)cxy.x, (double)cxy.y, A, B);
  // A, B, E decide the footprint edges (f64 -> f32 relative to rw0); invB and
  // cb only bound the candidate slices (0.01-slice margins): fp32 suffices
  const double Ar = A - (double)rw0;
  e.A = (float)Ar;
  e.B = (float)B;
  e.E = (float)(0.5 * B);
  e.invB = __frcp_rn(e.B);
  e.cb = (-0.5f - e.E - e.A) * e.invB - 0.01f;
}

// Band-specific part of an entry, evaluated by the lane that set the entry up:
// the slices za..zb that can reach rows [rw0, rw1], the staged range (za
// rounded down to a multiple of 4 for 16-byte loads), the 32-row groups the
// column's rows fall into, and whether the fast path applies.
__device__ __forceinline__ void band_info(FwEntry& e, const GridParams& gp, int rw0, int rw1, bool vec) {
  const int nc = cand_count(e.E, e.invB);
  const int za = max((int)floorf(fmaf((float)rw0, e.invB, e.cb)) + 1, 0);
  const int zb = min((int)floorf(fmaf((float)rw1, e.invB, e.cb)) + nc, gp.nz - 1);
  const int za4 = vec ? (za & ~3) : za;
  // rows reached by slices za..zb: [T(za) - E, T(zb) + E], widened by a row
  const float tlo = sub_(fma_(e.B, (float)za, e.A), e.E);
  const float thi = add_(fma_(e.B, (float)zb, e.A), e.E);
  const int r_lo = max((int)floorf(tlo) - 1, rw0), r_hi = min((int)ceilf(thi) + 1, rw1);
  const bool empty = za > zb || r_lo > r_hi;
  e.za4 = za4;
  e.nst = empty ? 0 : zb - za4 + 1;
  // x offset of the first staged slice, 32-bit: in float4 units on the vector
  // path (za4 and nz are multiples of 4), in floats otherwise; the launcher
  // checks nx*ny*nz < 2^34 resp. 2^32
  const unsigned xo = (unsigned)(((unsigned long long)(unsigned)e.col * (unsigned)gp.nz + (unsigned)za4) >> (vec ? 2 : 0));
  e.col = (int)xo;
  const int g0 = (r_lo - rw0) >> 5, g1 = (r_hi - rw0) >> 5;
  const bool fast = !empty && e.nst <= FW_XCAP && nc <= 3;
  e.info = empty ? 0 : (g0 | (g1 << 5) | (min(nc, 127) << 10) | (fast ? (1 << 17) : 0));
}

template <int NC>
__device__ __forceinline__ float fw_row_sum(const float* xs, float rf, float A, float B, float E, float invB,
                                            float cb, int off, int hic) {
  const float cf = floorf(fmaf(rf, invB, cb));  // first candidate - 1
  const int idx = min(max((int)cf + off, 0), hic);
  float rlo, rhi;  // r - .5, r + .5 (exact); volatile so they are formed per active row, not per entry
  asm volatile("{.reg .b64 ra, rd;\n\tmov.b64 ra, {%2, %2};\n\tadd.rn.f32x2 rd, ra, %3;\n\tmov.b64 {%0, %1}, rd;}"
               : "=f"(rlo), "=f"(rhi) : "f"(rf), "l"(0x3f000000bf000000ull));
  const float j0 = add_(cf, 1.0f);
  // The candidate window starts at most 0.99 slices past (r - .5 - E - A)/B
  // and ends at least 0.01 past (r + .5 + E - A)/B (E = B/2), so the first
  // candidate starts below the row (lo_0 < r - .5) and the last one ends above
  // it (hi_last > r + .5), each by >= 0.01 B rows, far beyond fp32 rounding:
  // max(lo_0, r - .5) is exactly r - .5 and min(hi_last, r + .5) exactly
  // r + .5, and only the other bounds are evaluated.
  const float2 T = fma2_(bc2_(B), make_float2(j0, add_(j0, 1.0f)), bc2_(A));
  float p;
  if (NC == 2) {
    const float2 hl = add2_(T, make_float2(E, -E));  // (hi_0, lo_1)
    float2 ov = add2_(make_float2(fminf(hl.x, rhi), rhi), make_float2(-rlo, -fmaxf(hl.y, rlo)));
    ov = make_float2(fmaxf(ov.x, 0.0f), fmaxf(ov.y, 0.0f));
    const float2 pp = mul2_(ov, make_float2(xs[idx], xs[idx + 1]));
    p = add_(pp.x, pp.y);
  } else {
    const float2 hi = add2_(T, bc2_(E));  // (hi_0, hi_1)
    const float lo1 = add_(T.y, -E);
    float2 ov = add2_(make_float2(fminf(hi.x, rhi), fminf(hi.y, rhi)), make_float2(-rlo, -fmaxf(lo1, rlo)));
    ov = make_float2(fmaxf(ov.x, 0.0f), fmaxf(ov.y, 0.0f));
    const float2 pp = mul2_(ov, make_float2(xs[idx], xs[idx + 1]));
    p = add_(pp.x, pp.y);
    const float T2 = fma_(B, add_(j0, 2.0f), A);
    const float lo2 = add_(T2, -E);
    const float o2 = fmaxf(sub_(rhi, fmaxf(lo2, rlo)), 0.0f);
    p = fma_(o2, xs[idx + 2], p);
  }
  return p;
}

#ifndef CTP_FW_PAIRS
#define CTP_FW_PAIRS 1  // each lane owns two adjacent rows; they share candidate slices
#endif
// Two adjacent rows r, r + 1 (row coordinate rf, rf + 1).  With two candidates
// per row (B >= 1.02), row r + 1's window starts d = 0 or 1 slices later, so
// the pair needs slices j0 .. j0 + 2 only: T, lo / hi and xa are evaluated once
// and row r + 1 selects its pair by d.  Every value is the one fw_row_sum<2>
// computes for that row (same fma / add operands), so results are bitwise
// unchanged.  Three candidates: two independent fw_row_sum<3> calls.
template <int NC>
__device__ __forceinline__ void fw_row_pair(const float* xs, float rf, float A, float B, float E, float invB,
                                            float cb, int off, int hic, float& pa, float& pb) {
  if (NC != 2) {
    pa = fw_row_sum<NC>(xs, rf, A, B, E, invB, cb, off, hic);
    pb = fw_row_sum<NC>(xs, add_(rf, 1.0f), A, B, E, invB, cb, off, hic);
    return;
  }
  const float rf1 = add_(rf, 1.0f);
  const float cfa = floorf(fmaf(rf, invB, cb));
  const float cfb = floorf(fmaf(rf1, invB, cb));
  const bool d = cfb > cfa;  // row r + 1's first candidate is j0 + 1
  const int idx = min(max((int)cfa + off, 0), hic);
  float rlo, rhi, rlo1, rhi1;
  asm volatile("{.reg .b64 ra, rd;\n\tmov.b64 ra, {%2, %2};\n\tadd.rn.f32x2 rd, ra, %3;\n\tmov.b64 {%0, %1}, rd;}"
               : "=f"(rlo), "=f"(rhi) : "f"(rf), "l"(0x3f000000bf000000ull));
  asm volatile("{.reg .b64 ra, rd;\n\tmov.b64 ra, {%2, %2};\n\tadd.rn.f32x2 rd, ra, %3;\n\tmov.b64 {%0, %1}, rd;}"
               : "=f"(rlo1), "=f"(rhi1) : "f"(rf1), "l"(0x3f000000bf000000ull));
  const float j0 = add_(cfa, 1.0f);
  const float2 T = fma2_(bc2_(B), make_float2(j0, add_(j0, 1.0f)), bc2_(A));
  const float T2 = fma_(B, add_(j0, 2.0f), A);
  const float2 hl = add2_(T, make_float2(E, -E));      // (hi_0, lo_1)
  const float2 hl1 = add2_(make_float2(T.y, T2), make_float2(E, -E));  // (hi_1, lo_2)
  const float x0 = xs[idx], x1 = xs[idx + 1], x2 = xs[idx + 2];
  float2 ov = add2_(make_float2(fminf(hl.x, rhi), rhi), make_float2(-rlo, -fmaxf(hl.y, rlo)));
  ov = make_float2(fmaxf(ov.x, 0.0f), fmaxf(ov.y, 0.0f));
  const float2 pp = mul2_(ov, make_float2(x0, x1));
  pa = add_(pp.x, pp.y);
  const float hf = d ? hl1.x : hl.x, ll = d ? hl1.y : hl.y;
  const float xf = d ? x1 : x0, xl = d ? x2 : x1;
  float2 ob = add2_(make_float2(fminf(hf, rhi1), rhi1), make_float2(-rlo1, -fmaxf(ll, rlo1)));
  ob = make_float2(fmaxf(ob.x, 0.0f), fmaxf(ob.y, 0.0f));
  const float2 pq = mul2_(ob, make_float2(xf, xl));
  pb = add_(pq.x, pq.y);
}

// Rows of this lane in the 32-row groups [g0, g1], FW_RG groups per step (one
// branch per block, so the independent row chains interleave; a row outside
// [g0, g1] inside an active block adds exactly 0):
// P(r) = sum over NC candidate slices j of tt(r, j) * xa(j), with T_j = A + B j
// recomputed in registers (the same fma as the back kernel, so lo/hi are
// bitwise equal) and only xa = amp * x staged in shared memory; then
// y(r, c) += ts(c) P(r).  tt = max(0, min(hi, r+.5) - max(lo, r-.5)) equals
// the back kernel's clamp(r+.5,lo,hi) - clamp(r-.5,lo,hi) bit for bit.
// Candidates outside the staged range read zero slots (idx is clamped to
// [0, hic]; both ends of the buffer hold >= 4 zeros, and a clamp only happens
// for virtual slices j < 0 or j >= nz, whose xa is 0).
#ifndef CTP_FW_RG
#if CTP_FW_PAIRS
#define CTP_FW_RG 2  // row slots evaluated per branch (one adjacent-row pair)
#else
#define CTP_FW_RG 3  // row groups evaluated per branch (independent chains that interleave)
#endif
#endif
constexpr int FW_RG = CTP_FW_RG;
static_assert(FW_KR % FW_RG == 0, "row groups are processed in blocks of FW_RG");

// row of register slot kk of this lane (lane's rbase = rw0 + lane, or
// rw0 + 2 lane with adjacent-row pairs)
__device__ __forceinline__ float fw_row_of(float rbase, int kk) {
#if CTP_FW_PAIRS
  return rbase + (float)(64 * (kk >> 1) + (kk & 1));
#else
  return rbase + (float)(32 * kk);
#endif
}
__device__ __forceinline__ int fw_row_base(int rw0, int lane) {
#if CTP_FW_PAIRS
  return rw0 + 2 * lane;
#else
  return rw0 + lane;
#endif
}

template <int NC>
__device__ __forceinline__ void fw_rows(float (&acc)[FW_KR][FW_CW], const float (&ts)[FW_CW],
                                        const float* xs, float rbase, float A, float B, float E,
                                        float invB, float cb, int off, int hic, int g0, int g1) {
#if CTP_FW_PAIRS
  static_assert(FW_RG % 2 == 0, "row pairs need an even FW_RG");
  g0 &= ~1;  // 32-row groups -> register slots: slot pair (2q, 2q+1) covers groups 2q, 2q+1
  g1 |= 1;
#endif
#pragma unroll
  for (int kk = 0; kk < FW_KR; kk += FW_RG) {
    if (kk + FW_RG - 1 < g0 || kk > g1) continue;  // warp-uniform
    float p[FW_RG];
#if CTP_FW_PAIRS
#pragma unroll
    for (int q = 0; q < FW_RG; q += 2)
      fw_row_pair<NC>(xs, fw_row_of(rbase, kk + q), A, B, E, invB, cb, off, hic, p[q], p[q + 1]);
#else
#pragma unroll
    for (int q = 0; q < FW_RG; ++q)
      p[q] = fw_row_sum<NC>(xs, fw_row_of(rbase, kk + q), A, B, E, invB, cb, off, hic);
#endif
#pragma unroll
    for (int cc = 0; cc < FW_CW; cc += 2) {
      const float2 t2 = make_float2(ts[cc], ts[cc + 1]);
#pragma unroll
      for (int q = 0; q < FW_RG; ++q) {
        const float2 a = fma2_(t2, bc2_(p[q]), make_float2(acc[kk + q][cc], acc[kk + q][cc + 1]));
        acc[kk + q][cc] = a.x;
        acc[kk + q][cc + 1] = a.y;
      }
    }
  }
}

// ---- warp-independent forward ------------------------------------------------
// One WARP owns one task = (view, FW_CW-column tile, FW_KR*32-row band).  It
// enumerates the wedge of voxel columns reaching its tile (rows of primary
// indices in chunks of 32, counts prefix-scanned with shuffles), sets the
// candidates up lane-parallel (one per lane, including everything the
// per-entry loop needs for this band), compacts the surviving (sub-)footprints
// into its private entry buffer, and gathers them into its register tile.  No
// CTA barriers: warps of a CTA never wait for each other.
#ifndef CTP_FV_WARPS
#define CTP_FV_WARPS 4
#endif
constexpr int FV_WARPS = CTP_FV_WARPS;
constexpr int FV_EBUF = 96;  // >= 31 pending + 64 from one setup round

#ifndef CTP_FW_CPASYNC
#define CTP_FW_CPASYNC 1  // prefetch x with cp.async into shared memory (vector path)
#endif
struct FvSmem {
  FwEntry ent[FV_EBUF];
  float xs[FW_XLEN];  // staged amp * x of one entry (or one piece)
#if CTP_FW_CPASYNC
  float xr[2][FW_XCAP];  // raw x of the next fast entries, filled by cp.async
#endif
};

size_t forward_warp_smem_bytes() { return sizeof(FvSmem) * FV_WARPS; }

// issue the loads of x for the staged slices of one entry (16-byte loads when
// the column layout allows, slots >= nst read as 0)
template <bool VEC>
__device__ __forceinline__ void fw_prefetch(float4 (&xv)[FW_NLD], const float* __restrict__ xc, int nst,
                                            int lane) {
#pragma unroll
  for (int t = 0; t < FW_NLD; ++t) {
    const int s = 4 * lane + 128 * t;
    if (VEC) {
      // slots >= nst are never staged: clamp to the last (valid) float4 instead of predicating
      xv[t] = __ldg(reinterpret_cast<const float4*>(xc + min(s, (nst - 1) & ~3)));
    } else {
      xv[t].x = s < nst ? __ldg(xc + s) : 0.0f;
      xv[t].y = s + 1 < nst ? __ldg(xc + s + 1) : 0.0f;
      xv[t].z = s + 2 < nst ? __ldg(xc + s + 2) : 0.0f;
      xv[t].w = s + 3 < nst ? __ldg(xc + s + 3) : 0.0f;
    }
  }
}

template <bool VEC>
__device__ __forceinline__ void fw_process(FvSmem& S, int nent, float (&acc)[FW_KR][FW_CW],
                                           const GridParams& gp, const float* __restrict__ xb,
                                           int rw0, int lane) {
  float* xs = S.xs;
  const float rbase = (float)fw_row_base(rw0, lane);  // rw0 = 0: rows relative to the band
  // software pipeline: x of the next fast-path entry is in flight while the
  // current entry is gathered
  constexpr bool ASYNC = VEC && CTP_FW_CPASYNC;
#if CTP_FW_CPASYNC
  int pbuf = 0;  // xr buffer the next prefetch goes to
#endif
  float4 xv[FW_NLD];  // (register prefetch; unused, hence free, on the cp.async path)
  auto next_fast = [&](int e) {
    for (; e < nent; ++e) {
      if (S.ent[e].info & (1 << 17)) {
        const float* xc = xb + ((size_t)(unsigned)S.ent[e].col << (VEC ? 2 : 0));
#if CTP_FW_CPASYNC
        if constexpr (ASYNC) {
          const int nst = S.ent[e].nst;
#pragma unroll
          for (int t = 0; t < FW_NLD; ++t) {
            const int s = 4 * lane + 128 * t;
            if (s < nst) cp_async16(&S.xr[pbuf][s], xc + s);
          }
          cp_async_commit();
          pbuf ^= 1;
          return e;
        }
#endif
        fw_prefetch<VEC>(xv, xc, S.ent[e].nst, lane);
        return e;
      }
    }
    return nent;
  };
  int e_pf = next_fast(0);
  for (int e = 0; e < nent; ++e) {
    const FwEntry& E = S.ent[e];
    const int info = E.info;
    const int nst = E.nst;
    if (nst == 0) continue;
    const float A = E.A, B = E.B, Eh = E.E, lxy = E.lxy, a0 = E.a0, a1 = E.a1;
    const float invB = E.invB, cb = E.cb;
    const int za4 = E.za4;
    const int g0 = info & 31, g1 = (info >> 5) & 31, nc = (info >> 10) & 127;
    float ts[FW_CW];
#pragma unroll
    for (int cc = 0; cc < FW_CW; ++cc) ts[cc] = E.ts[cc];
    if (e == e_pf) {
#if CTP_FW_CPASYNC
      const float* xraw = nullptr;
      if constexpr (ASYNC) {
        cp_async_wait_all();  // this lane's copies; the warp barrier publishes the others'
        __syncwarp();
        xraw = S.xr[pbuf ^ 1];
      }
#endif
      // stage xa = amp * x of slices za4 .. za4 + nst - 1 (4 per lane and load),
      // FW_SG loads per branch so their chains interleave
#pragma unroll
      for (int t0 = 0; t0 < FW_NLD; t0 += FW_SG) {
        if (128 * t0 >= nst) break;  // warp-uniform
#pragma unroll
        for (int t = t0; t < t0 + FW_SG; ++t) {
          const int s = 4 * lane + 128 * t;
          const float z0 = (float)(za4 + s);
          const float2 izA = make_float2(z0, add_(z0, 1.0f)), izB = make_float2(add_(z0, 2.0f), add_(z0, 3.0f));
          const float2 qA = fma2_(bc2_(a1), izA, bc2_(a0)), qB = fma2_(bc2_(a1), izB, bc2_(a0));
          const float2 tA = fma2_(qA, qA, bc2_(1.0f)), tB = fma2_(qB, qB, bc2_(1.0f));
          const float2 ampA = mul2_(bc2_(lxy), make_float2(sqrt_approx(tA.x), sqrt_approx(tA.y)));
          const float2 ampB = mul2_(bc2_(lxy), make_float2(sqrt_approx(tB.x), sqrt_approx(tB.y)));
          float4 xq;
#if CTP_FW_CPASYNC
          if constexpr (ASYNC) xq = *reinterpret_cast<const float4*>(xraw + s);
          else
#endif
            xq = xv[t];
          const float2 xaA = mul2_(ampA, make_float2(xq.x, xq.y));
          const float2 xaB = mul2_(ampB, make_float2(xq.z, xq.w));
          if (s < nst) *reinterpret_cast<float4*>(xs + FW_XPAD + s) = make_float4(xaA.x, xaA.y, xaB.x, xaB.y);
        }
      }
      if (lane < 4) xs[FW_XPAD + ((nst + 3) & ~3) + lane] = 0.0f;
      __syncwarp();
      e_pf = next_fast(e + 1);  // loads for the next entry overlap this gather
      const int off = 1 - za4 + FW_XPAD, hic = FW_XPAD + nst;
      if (nc <= 2) fw_rows<2>(acc, ts, xs, rbase, A, B, Eh, invB, cb, off, hic, g0, g1);
      else fw_rows<3>(acc, ts, xs, rbase, A, B, Eh, invB, cb, off, hic, g0, g1);
      __syncwarp();
      continue;
    }
    // generic path: many candidates per row and/or more slices than one
    // staging buffer holds; pieces of FW_XCAP slices, exact candidate loops
    const int za = max((int)floorf(fmaf((float)rw0, invB, cb)) + 1, 0);
    const int zb = za4 + nst - 1;
    float P[FW_KR];
#pragma unroll
    for (int kk = 0; kk < FW_KR; ++kk) P[kk] = 0.0f;
    const float* xc = xb + (((size_t)(unsigned)E.col << (VEC ? 2 : 0)) - za4);
    for (int piece = za; piece <= zb; piece += FW_XCAP) {
      const int pe = min(piece + FW_XCAP - 1, zb);
      const int n = pe - piece + 1;
      for (int i = lane; i < n; i += 32) {
        const float izf = (float)(piece + i);
        const float q = fma_(a1, izf, a0);
        const float amp = mul_(lxy, sqrt_approx(fma_(q, q, 1.0f)));
        xs[FW_XPAD + i] = mul_(amp, __ldg(xc + piece + i));
      }
      __syncwarp();
#if CTP_FW_PAIRS
      const int k0 = g0 & ~1, k1 = g1 | 1;
#else
      const int k0 = g0, k1 = g1;
#endif
#pragma unroll
      for (int kk = 0; kk < FW_KR; ++kk) {
        if (kk < k0 || kk > k1) continue;
        const float rf = fw_row_of(rbase, kk);
        const float rlo = sub_(rf, 0.5f), rhi = add_(rf, 0.5f);
        const int c = (int)floorf(fmaf(rf, invB, cb));
        const int j1 = min(c + nc, pe);
        float p = P[kk];
        for (int j = max(c + 1, piece); j <= j1; ++j) {
          const float T = fma_(B, (float)j, A);
          const float lo = add_(T, -Eh), hi = add_(T, Eh);
          p = fma_(fmaxf(sub_(fminf(hi, rhi), fmaxf(lo, rlo)), 0.0f), xs[FW_XPAD + j - piece], p);
        }
        P[kk] = p;
      }
      __syncwarp();
    }
#pragma unroll
    for (int kk = 0; kk < FW_KR; ++kk)
#pragma unroll
      for (int cc = 0; cc < FW_CW; ++cc) acc[kk][cc] = fma_(ts[cc], P[kk], acc[kk][cc]);
  }
}

// Footprint setup of the wedge candidates k = cbase + lane (one per lane):
// owner primary index by binary search over the exclusive scan, footprint of
// the voxel column, test against the tile, compaction of the surviving
// (sub-)footprints into ent[0..).  Returns how many entries the warp added.
// Out of line: it holds most of the kernel's geometry, and keeping it out of
// the gather loop's register allocation avoids rematerialisation there.
__device__ __noinline__ int fw_candidates(const GridParams& gp, const ViewCoef* __restrict__ vcp,
                                          const ViewAx* __restrict__ vaxp, FwEntry* ent, int k, int total, int ib,
                                          int excl, int jl, bool primary_x, int c0, int cw, float band_lo,
                                          float band_hi, int rw0, int rw1, bool vec) {
  const int lane = threadIdx.x & 31;
  // owner lane o: the largest lane with excl_o <= k (it has cnt_o > 0)
  int o = 0;
#pragma unroll
  for (int step = 16; step >= 1; step >>= 1) {
    const int ex = __shfl_sync(0xffffffffu, excl, o + step);
    if (ex <= k) o += step;
  }
  const int jo = __shfl_sync(0xffffffffu, jl, o);
  const int exo = __shfl_sync(0xffffffffu, excl, o);
  SubFoot f0, f1;
  float2 cxy0 = make_float2(0.0f, 0.0f), cxy1 = cxy0;
  int mask = 0, col = 0;
  if (k < total) {
    const ViewCoef vc = *vcp;
    const int ii = ib + o, j = jo + (k - exo);
    const int ix = primary_x ? ii : j, iy = primary_x ? j : ii;
    col = iy * gp.nx + ix;
    mask = column_subs(vc, gp, ix, iy, f0, f1, cxy0, cxy1) & 3;
    if ((mask & 1) && !reaches_tile(f0, gp, c0, cw, band_lo, band_hi)) mask &= ~1;
    if ((mask & 2) && !reaches_tile(f1, gp, c0, cw, band_lo, band_hi)) mask &= ~2;
  }
  const int n = __popc(mask);
  const int ni = warp_incl_scan(n, lane);
  const int off = ni - n;
  if (mask & 1) {
    write_entry(ent[off], f0, col, c0, cw);
    localize_entry(ent[off], *vaxp, gp, cxy0, rw0);
    band_info(ent[off], gp, 0, rw1 - rw0, vec);
  }
  if (mask & 2) {
    write_entry(ent[off + (mask & 1)], f1, col, c0, cw);
    localize_entry(ent[off + (mask & 1)], *vaxp, gp, cxy1, rw0);
    band_info(ent[off + (mask & 1)], gp, 0, rw1 - rw0, vec);
  }
  return __shfl_sync(0xffffffffu, ni, 31);
}

template <bool VEC>
__global__ void __launch_bounds__(FV_WARPS * 32, CTP_FW_MINB) sf_forward_kernel(
    const __grid_constant__ GridParams gp, const ViewCoef* __restrict__ vcoef, const ViewAx* __restrict__ vax,
    const float* __restrict__ xT, float* __restrict__ y, int accumulate, long long task0, long long ntasks) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  FvSmem& S = reinterpret_cast<FvSmem*>(smem_raw)[warp];
  const long long task = task0 + (long long)blockIdx.x * FV_WARPS + warp;
  if (task >= ntasks) return;  // warp-uniform; no CTA barriers in this kernel
  const int ntiles = (gp.nc + FW_CW - 1) / FW_CW;
  // band-major task order: consecutive CTAs sweep views and tiles of one row
  // band, i.e. the same z-range of the volume, which then stays in L2
  const long long per_band = (long long)ntiles * gp.nv * gp.batch;
  const int band = (int)(task / per_band);
  const long long t2 = task % per_band;
#if CTP_FW_VCH > 0
  // within a band: chunks of FW_VCH consecutive views, tiles, views of the
  // chunk -- the CTAs resident at once cover a few dozen adjacent tiles over a
  // few degrees of rotation, whose wedges (a fraction of the volume) stay in L2
  const int nvb = gp.nv * gp.batch;
  const int vch = (int)(t2 / ((long long)ntiles * FW_VCH));
  const int rem = (int)(t2 - (long long)vch * ntiles * FW_VCH);
  const int cv = min(FW_VCH, nvb - vch * FW_VCH);
  const int tile = rem / cv;
  const int vb = vch * FW_VCH + rem % cv;
#else
  const int tile = (int)(t2 % ntiles);
  const int vb = (int)(t2 / ntiles);
#endif
  const int v = vb % gp.nv, b = vb / gp.nv;
  const int c0 = tile * FW_CW;
  const int cw = min(FW_CW, gp.nc - c0);
  const int rw0 = band * FW_ROWS;
  const int rw1 = min(rw0 + FW_ROWS, gp.nr) - 1;
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
  const float band_lo = (float)rw0 - 0.5f, band_hi = (float)rw1 + 0.5f;

  float acc[FW_KR][FW_CW];
#pragma unroll
  for (int k = 0; k < FW_KR; ++k)
#pragma unroll
    for (int c = 0; c < FW_CW; ++c) acc[k][c] = 0.0f;
  if (lane < FW_XPAD) S.xs[lane] = 0.0f;  // zero slots below the staged slices
  __syncwarp();
  const float* xb = xT + (size_t)b * ((size_t)gp.nx * gp.ny) * gp.nz;

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
      pending += fw_candidates(gp, vcoef + v, vax + v, S.ent + pending, cbase + lane, total, ib, excl, jl, primary_x,
                               c0, cw, band_lo, band_hi, rw0, rw1, VEC);
      __syncwarp();
      if (pending >= 32) {
        fw_process<VEC>(S, pending, acc, gp, xb, 0, lane);
        pending = 0;
        __syncwarp();
      }
    }
  }
  if (pending > 0) fw_process<VEC>(S, pending, acc, gp, xb, 0, lane);

  // store the tile: y[b][v][r][c0 + c]
  float* yv = y + ((size_t)b * gp.nv + v) * (size_t)gp.nr * gp.nc;
#pragma unroll
  for (int kk = 0; kk < FW_KR; ++kk) {
    const int r = (int)fw_row_of((float)fw_row_base(rw0, lane), kk);
    if (r > rw1) continue;
    float* row = yv + (size_t)r * gp.nc + c0;
#pragma unroll
    for (int c = 0; c < FW_CW; ++c) {
      if (c >= cw) break;
      row[c] = accumulate ? row[c] + acc[kk][c] : acc[kk][c];
    }
  }
}

// ---------------------------------------------------------------------------
// fan beam (one slice, one detector row) with the batch on the lanes
// ---------------------------------------------------------------------------
// BASELINE configs[1]: 64 slices share one geometry, so one footprint setup
// serves the whole batch.  Layouts are batch-innermost ([pixel][B] volumes,
// [v][c][B] sinograms, produced by transpose_kernel) so the lanes of a warp
// (consecutive batch elements) read and write consecutive addresses.  The
// coefficient association is the same as in the 3D pair:
//   forward  y += ts * (tt * (amp * x)),   back  x += (amp * tt) * (sum ts * y).
constexpr int F2_MAXG = 4;  // batch groups of 32 per warp (batch <= 128 per launch)

// axial weight of detector row 0 for slice iz = 0 (boundary rule of the 3D pair)
__device__ __forceinline__ float row0_weight(float A, float B, float E, bool& hit) {
  const float T = fma_(B, 0.0f, A);
  const float lo = add_(T, -E), hi = add_(T, E);
  const float fl = floorf(add_(lo, -0.5f));
  const int K = rows_per_slice(B);
  const int k = -((int)fl + 1);  // row 0 = r0 + k
  hit = k >= 0 && k < K;
  if (!hit) return 0.0f;
  const float lower = (k == 0) ? lo : clampf_(add_(fl, (float)k + 0.5f), lo, hi);
  const float upper = (k == K - 1) ? hi : clampf_(add_(fl, (float)k + 1.5f), lo, hi);
  return add_(upper, -lower);
}

#ifndef CTP_FB_ALONG_Y
#define CTP_FB_ALONG_Y 1
#endif
template <int G>
__global__ void __launch_bounds__(256) sf_back_fan_kernel(GridParams gp, const ViewCoef* __restrict__ vcoef,
                                                          const float* __restrict__ yB,  // [nv][nc][Bs]
                                                          float* __restrict__ xo,        // [Bs][ny*nx]
                                                          int Bs, int b0, int nb) {
  __shared__ __align__(16) BkEntry ents[8][32][2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#if CTP_FB_ALONG_Y
  // the CTA's 8 warps: 8 consecutive pixels along y (shared detector columns)
  const int ix = blockIdx.x % gp.nx, iy = (blockIdx.x / gp.nx) * 8 + warp;
  if (iy >= gp.ny) return;
  const int pix = iy * gp.nx + ix;
#else
  const int pix = blockIdx.x * 8 + warp;
  if (pix >= gp.nx * gp.ny) return;
  const int ix = pix % gp.nx, iy = pix / gp.nx;
#endif
  BkEntry(&my)[32][2] = ents[warp];
  float acc[G];
#pragma unroll
  for (int g = 0; g < G; ++g) acc[g] = 0.0f;
  const size_t view_stride = (size_t)gp.nc * Bs;
  for (int vb = 0; vb < gp.nv; vb += 32) {
    const int nsub = back_setup(gp, vcoef, vb, ix, iy, 0, 0, &my[lane][0]) ? 2 : 1;
    // lane-parallel: the view's axial weight of row 0 times the amplitude,
    // c = amp * tt (the 3D kernels' (amp * tt) factor), kept in the entry's
    // lxy slot; entries that miss row 0 are dropped
    bool narrow = true;  // no footprint wider than BK_NCF columns in this batch
    for (int s = 0; s < nsub; ++s) {
      BkEntry& e = my[lane][s];
      bool hit = false;
      const float tt = e.ncol > 0 ? row0_weight(e.A, e.B, e.E, hit) : 0.0f;
      const float amp = mul_(e.lxy, sqrt_approx(fma_(e.a0, e.a0, 1.0f)));
      if (!hit) e.ncol = 0;
      if (e.ncol <= BK_NCF) {
        // narrow: c = amp * tt, and a column window cl..cl+3 inside the
        // detector whose weights outside the footprint are 0 (each adds an
        // exact 0); missing entries get c = 0
        e.lxy = e.ncol > 0 ? mul_(amp, tt) : 0.0f;
        const int cl = min(e.ncol > 0 ? e.cl : 0, max(gp.nc - BK_NCF, 0));
        float t[BK_NCF];
#pragma unroll
        for (int k = 0; k < BK_NCF; ++k) {
          const int kk = cl + k - e.cl;  // index of column cl + k in the footprint's weights
          t[k] = 0.0f;
#pragma unroll
          for (int m = 0; m < BK_NCF; ++m)
            if (kk == m && m < e.ncol) t[k] = e.ts[m];
        }
#pragma unroll
        for (int k = 0; k < BK_NCF; ++k) e.ts[k] = t[k];
        e.cl = cl;
      } else {
        narrow = false;
      }
    }
    narrow = __all_sync(0xffffffffu, narrow) && gp.nc >= BK_NCF;
    __syncwarp();
    const int nvb = min(32, gp.nv - vb);
    const float* yview = yB + (size_t)vb * view_stride + b0;
    if (narrow && nsub == 1) {
      // every entry of the batch is a narrow window: branch-free, unrolled
      // over views so loads of consecutive views overlap
#pragma unroll 4
      for (int j = 0; j < nvb; ++j) {
        const BkEntry& e = my[j][0];
        const float c = e.lxy;
        const float* yc = yview + (size_t)j * view_stride + (size_t)e.cl * Bs;
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const int b = lane + 32 * g;
          if (b >= nb) break;
          float q = mul_(e.ts[0], __ldg(yc + b));
#pragma unroll
          for (int k = 1; k < BK_NCF; ++k) q = fma_(e.ts[k], __ldg(yc + (size_t)k * Bs + b), q);
          acc[g] = fma_(c, q, acc[g]);
        }
      }
      __syncwarp();
      continue;
    }
    for (int j = 0; j < nvb; ++j, yview += view_stride) {
#pragma unroll 1
      for (int s = 0; s < nsub; ++s) {
        const BkEntry& e = my[j][s];
        const int ncol = e.ncol;
        if (ncol == 0) continue;
        if (ncol <= BK_NCF) {
          const float c = e.lxy;
          const float* yc = yview + (size_t)e.cl * Bs;
          float t4[BK_NCF];
#pragma unroll
          for (int k = 0; k < BK_NCF; ++k) t4[k] = e.ts[k];
#pragma unroll
          for (int g = 0; g < G; ++g) {
            const int b = lane + 32 * g;
            if (b >= nb) break;
            float q = mul_(t4[0], __ldg(yc + b));
#pragma unroll
            for (int k = 1; k < BK_NCF; ++k) q = fma_(t4[k], __ldg(yc + (size_t)k * Bs + b), q);  // (window)
            acc[g] = fma_(c, q, acc[g]);
          }
          continue;
        }
        // wide footprint (> BK_NCF columns): rebuild its breakpoints
        bool hit;
        const float tt = row0_weight(e.A, e.B, e.E, hit);
        const float c = mul_(mul_(e.lxy, sqrt_approx(fma_(e.a0, e.a0, 1.0f))), tt);
        SubFoot f0, f1;
        column_footprint(vcoef[vb + j], gp, ix, iy, f0, f1);
        const Trap wide = make_trap(s == 0 ? f0 : f1);
        for (int g = 0; g < G; ++g) {
          const int b = lane + 32 * g;
          if (b >= nb) break;
          float q = 0.0f;
          float prev = trap_cum(wide, sub_((float)e.cl, 0.5f));
          for (int k = 0; k < ncol; ++k) {
            const float cur = trap_cum(wide, add_((float)(e.cl + k), 0.5f));
            q = fma_(sub_(cur, prev), __ldg(yview + (size_t)(e.cl + k) * Bs + b), q);
            prev = cur;
          }
          acc[g] = fma_(c, q, acc[g]);
        }
      }
    }
    __syncwarp();
  }
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int b = lane + 32 * g;
    // natural layout out[b][iy][ix] (lane stride ny*nx: one 4-byte store per
    // lane, but no batch-innermost copy of the volume in the workspace)
    if (b < nb) xo[(size_t)(b0 + b) * ((size_t)gp.nx * gp.ny) + pix] = acc[g];
  }
}

// Fan-beam variant of fw_candidates: the footprint of candidate k = cbase +
// lane, its tile test, and the fan-specific per-entry factors (axial weight
// of row 0 in a1, amplitude in lxy), compacted into ent[0..); entries that
// miss row 0 are dropped.  Out of line for the same register reasons.
__device__ __noinline__ int fan_candidates(const GridParams& gp, const ViewCoef* __restrict__ vcp, FwEntry* ent,
                                           int k, int total, int ib, int excl, int jl, bool primary_x, int c0,
                                           int cw, float band_lo, float band_hi) {
  const int lane = threadIdx.x & 31;
  int o = 0;
#pragma unroll
  for (int step = 16; step >= 1; step >>= 1) {
    const int ex = __shfl_sync(0xffffffffu, excl, o + step);
    if (ex <= k) o += step;
  }
  const int jo = __shfl_sync(0xffffffffu, jl, o);
  const int exo = __shfl_sync(0xffffffffu, excl, o);
  SubFoot f[2];
  float tt[2] = {0.0f, 0.0f};
  int mask = 0, col = 0;
  if (k < total) {
    const ViewCoef vc = *vcp;
    const int ii = ib + o, j = jo + (k - exo);
    const int ix = primary_x ? ii : j, iy = primary_x ? j : ii;
    col = iy * gp.nx + ix;
    mask = column_footprint(vc, gp, ix, iy, f[0], f[1]);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      if (!(mask & (1 << h))) continue;
      bool hit = false;
      if (reaches_tile(f[h], gp, c0, cw, band_lo, band_hi)) tt[h] = row0_weight(f[h].A, f[h].B, f[h].E, hit);
      if (!hit) mask &= ~(1 << h);
    }
  }
  const int n = __popc(mask);
  const int ni = warp_incl_scan(n, lane);
  int off = ni - n;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (!(mask & (1 << h))) continue;
    FwEntry& e = ent[off++];
    write_entry(e, f[h], col, c0, cw);
    e.a1 = tt[h];
    e.lxy = mul_(f[h].lxy, sqrt_approx(fma_(f[h].a0, f[h].a0, 1.0f)));  // amp at iz = 0
  }
  return __shfl_sync(0xffffffffu, ni, 31);
}

#ifndef CTP_FF_VIEWS_FAST
#define CTP_FF_VIEWS_FAST 1
#endif
template <int G>
__global__ void __launch_bounds__(FV_WARPS * 32) sf_forward_fan_kernel(
    const __grid_constant__ GridParams gp, const ViewCoef* __restrict__ vcoef, const float* __restrict__ xB,  // [ny*nx][Bs]
    float* __restrict__ yo,                                                         // [Bs][nv][nc]
    int Bs, int b0, int nb) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  FwEntry* ent = reinterpret_cast<FwEntry*>(smem_raw) + warp * FV_EBUF;
  const int ntiles = (gp.nc + FW_CW - 1) / FW_CW;
  const long long task = (long long)blockIdx.x * FV_WARPS + warp;
  if (task >= (long long)ntiles * gp.nv) return;
#if CTP_FF_VIEWS_FAST
  // consecutive warps: the same tile in consecutive views (their wedges, and
  // the pixels' batch rows they read, nearly coincide -> L1 reuse)
  const int tile = (int)(task / gp.nv);
  const int v = (int)(task % gp.nv);
#else
  const int tile = (int)(task % ntiles);
  const int v = (int)(task / ntiles);
#endif
  const int c0 = tile * FW_CW;
  const int cw = min(FW_CW, gp.nc - c0);
  const ViewCoef vc = vcoef[v];
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

  float acc[G][FW_CW];
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int c = 0; c < FW_CW; ++c) acc[g][c] = 0.0f;

  int pending = 0;
  auto flush = [&]() {
#pragma unroll 2
    for (int e = 0; e < pending; ++e) {
      const FwEntry& E = ent[e];
      const float tt = E.a1, amp = E.lxy;  // set up by fan_candidates
      const float* xc = xB + (size_t)E.col * Bs + b0;
      float ts[FW_CW];
#pragma unroll
      for (int cc = 0; cc < FW_CW; ++cc) ts[cc] = E.ts[cc];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const int b = lane + 32 * g;
        const float xv = b < nb ? __ldg(xc + b) : 0.0f;
        const float P = mul_(tt, mul_(amp, xv));
        const float2 pp = bc2_(P);
#pragma unroll
        for (int cc = 0; cc < FW_CW; cc += 2) {
          const float2 a = fma2_(make_float2(ts[cc], ts[cc + 1]), pp, make_float2(acc[g][cc], acc[g][cc + 1]));
          acc[g][cc] = a.x;
          acc[g][cc + 1] = a.y;
        }
      }
    }
    pending = 0;
  };
  const float band_lo = -0.5f, band_hi = (float)gp.nr - 0.5f;
  for (int ib = 0; ib < nP; ib += 32) {
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
      pending += fan_candidates(gp, vcoef + v, ent + pending, cbase + lane, total, ib, excl, jl, primary_x, c0,
                                cw, band_lo, band_hi);
      __syncwarp();
      if (pending >= 32) {
        flush();
        __syncwarp();
      }
    }
  }
  if (pending > 0) flush();
  // natural layout y[b][v][c0 .. c0 + 3] (16 contiguous bytes per lane, no
  // batch-innermost copy of the sinogram in the workspace)
  float* yv = yo + (size_t)v * gp.nc + c0;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const int b = lane + 32 * g;
    if (b >= nb) continue;
#pragma unroll
    for (int c = 0; c < FW_CW; ++c)
      if (c < cw) yv[(size_t)(b0 + b) * gp.nv * gp.nc + c] = acc[g][c];
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
cudaError_t launch_transpose(const float* in, float* out, int R, int C, int batch,
                             cudaStream_t st) {
  const dim3 block(256);
  for (int b0 = 0; b0 < batch; b0 += 65535) {
    const int nb = min(65535, batch - b0);
    // row blocks in launches of <= 65535 (gridDim.y limit): large fan sinograms
    // and slices (nv*nc or nx*ny above ~2.1M elements) need several
    const int nrb = (R + 31) / 32;
    for (int rb0 = 0; rb0 < nrb; rb0 += 65535) {
      const dim3 grid((C + 31) / 32, min(65535, nrb - rb0), nb);
      transpose_kernel<<<grid, block, 0, st>>>(in, out, R, C, b0, rb0);
    }
  }
  return cudaGetLastError();
}

cudaError_t launch_back_legacy(const GridParams& gp, const ViewCoef* vcoef, const ViewAx* vax, const float* yT,
                               float* vol, int batch, bool accumulate, cudaStream_t st, int z0, int z1) {
  if (z1 < 0) z1 = gp.nz;
  if (z0 < 0 || z0 >= z1 || z1 > gp.nz) return cudaErrorInvalidValue;
  cudaError_t ea = cudaFuncSetAttribute(sf_back_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)sizeof(BkSmem));
  if (ea != cudaSuccess) return ea;
  const int nbx = (gp.nx + BK_CX - 1) / BK_CX, nby = (gp.ny + BK_WARPS / BK_CX - 1) / (BK_WARPS / BK_CX);
  for (int b0 = 0; b0 < batch; b0 += 65535) {
    const int nb = min(65535, batch - b0);
    const dim3 grid(nbx * nby, (z1 - z0 + BK_ZC - 1) / BK_ZC, nb);
    const size_t sino_elems = (size_t)gp.nv * gp.nr * gp.nc;
    const size_t vol_elems = (size_t)gp.nx * gp.ny * gp.nz;
    sf_back_kernel<<<grid, BK_WARPS * 32, sizeof(BkSmem), st>>>(gp, vcoef, vax, yT + (size_t)b0 * sino_elems,
                                                                vol + (size_t)b0 * vol_elems, accumulate ? 1 : 0,
                                                                z0, z1);
  }
  return cudaGetLastError();
}

cudaError_t launch_forward_legacy(const GridParams& gp, const ViewCoef* vcoef, const ViewAx* vax, const float* xT,
                                  float* sino, int batch, bool accumulate, cudaStream_t st) {
  const size_t smem = forward_warp_smem_bytes();
  // 16-byte x loads need every voxel column (nz floats) 16-byte aligned
  const bool vec = gp.nz % 4 == 0 && (reinterpret_cast<uintptr_t>(xT) & 15) == 0;
  // 32-bit x offsets per entry (float4 units on the vector path)
  if ((long long)gp.nx * gp.ny * gp.nz >= (vec ? (1LL << 34) : (1LL << 32))) return cudaErrorInvalidValue;
  auto kern = vec ? sf_forward_kernel<true> : sf_forward_kernel<false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const long long nbands = (gp.nr + FW_ROWS - 1) / FW_ROWS;
  const long long ntiles = (gp.nc + FW_CW - 1) / FW_CW;
  const long long ntasks = nbands * ntiles * (long long)gp.nv * batch;
  const long long max_blocks = 1LL << 30;
  GridParams g2 = gp;
  g2.batch = batch;  // the task decode needs the batch extent
  for (long long t0 = 0; t0 < ntasks; t0 += max_blocks * FV_WARPS) {
    const long long rem = ntasks - t0;
    const long long nb = (rem + FV_WARPS - 1) / FV_WARPS;
    const unsigned grid = (unsigned)(nb < max_blocks ? nb : max_blocks);
    kern<<<grid, FV_WARPS * 32, smem, st>>>(g2, vcoef, vax, xT, sino, accumulate ? 1 : 0, t0, ntasks);
  }
  return cudaGetLastError();
}

// xB: [ny*nx][batch] (batch-innermost input); sino: [batch][nv][nc]; nz == nr == 1
cudaError_t launch_forward_fan(const GridParams& gp, const ViewCoef* vcoef, const float* xB, float* sino,
                               int batch, cudaStream_t st) {
  const size_t smem = sizeof(FwEntry) * FV_EBUF * FV_WARPS;
  const long long ntasks = (long long)((gp.nc + FW_CW - 1) / FW_CW) * gp.nv;
  const unsigned grid = (unsigned)((ntasks + FV_WARPS - 1) / FV_WARPS);
  for (int b0 = 0; b0 < batch; b0 += 32 * F2_MAXG) {
    const int nb = min(32 * F2_MAXG, batch - b0);
    const int G = (nb + 31) / 32;
    cudaError_t e = cudaSuccess;
#define CTP_FAN_FWD(g)                                                                              \
  case g:                                                                                           \
    e = cudaFuncSetAttribute(sf_forward_fan_kernel<g>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             (int)smem);                                                            \
    if (e != cudaSuccess) return e;                                                                 \
    sf_forward_fan_kernel<g><<<grid, FV_WARPS * 32, smem, st>>>(gp, vcoef, xB, sino, batch, b0, nb); \
    break;
    switch (G) { CTP_FAN_FWD(1) CTP_FAN_FWD(2) CTP_FAN_FWD(3) default: CTP_FAN_FWD(4) }
#undef CTP_FAN_FWD
  }
  return cudaGetLastError();
}

cudaError_t launch_back_fan(const GridParams& gp, const ViewCoef* vcoef, const float* yB, float* vol,
                            int batch, cudaStream_t st) {
#if CTP_FB_ALONG_Y
  const unsigned grid = (unsigned)(gp.nx * ((gp.ny + 7) / 8));
#else
  const unsigned grid = (unsigned)((gp.nx * gp.ny + 7) / 8);
#endif
  for (int b0 = 0; b0 < batch; b0 += 32 * F2_MAXG) {
    const int nb = min(32 * F2_MAXG, batch - b0);
    const int G = (nb + 31) / 32;
    switch (G) {
      case 1: sf_back_fan_kernel<1><<<grid, 256, 0, st>>>(gp, vcoef, yB, vol, batch, b0, nb); break;
      case 2: sf_back_fan_kernel<2><<<grid, 256, 0, st>>>(gp, vcoef, yB, vol, batch, b0, nb); break;
      case 3: sf_back_fan_kernel<3><<<grid, 256, 0, st>>>(gp, vcoef, yB, vol, batch, b0, nb); break;
      default: sf_back_fan_kernel<4><<<grid, 256, 0, st>>>(gp, vcoef, yB, vol, batch, b0, nb); break;
    }
  }
  return cudaGetLastError();
}

}  // namespace ctp
