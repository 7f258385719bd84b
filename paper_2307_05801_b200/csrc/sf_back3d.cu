// sf_back3d.cu -- 3D back projection x = A^T y of the SF-TR pair (parallel,
// cone flat/curved, SF-modular), voxel-driven GATHER (reference:
// sf_back_kernel, _kernels.py:666-763).
//
// Integral formulation.  For one voxel column (ix, iy) in one view the axial
// footprints of consecutive slices TILE the detector column: slice i spans
// rows [W0 + B i, W0 + B (i + 1)) (row units, B = mag hz / ph), so
//
//   x[i] += amp_i * sum_r overlap(slice i, row r) * Q(r),   Q(r) = sum_c ts(c) y[c][r]
//         = amp_i * (H(w_{i+1}) - H(w_i)),
//
// where H is the integral of the piecewise-constant row profile Q:
// H(w) = S_k + (w - k) Q_k, k = floor(w), S_k = sum_{j<k} Q_j.  The reference
// sums tt(r) Q(r) over the 2-3 rows a slice touches (_kernels.py:738-760);
// here a warp builds the running sums of Q over the rows its slices reach
// once per view and every slice costs ONE table evaluation: lanes own slices
// lane + 32 m, each lane evaluates H at the upper boundary of its slice and
// takes the lower one from lane - 1 with a shuffle.  The input stage
// (sino_prefix.cu) hands the kernel per-column prefix sums over aligned
// 128-row segments, so a table is a weighted sum of those (coalesced 16-byte
// loads along the row-contiguous sinogram) plus one carry per segment: no
// warp scans.  Mathematically identical to the reference; in fp32 the prefix
// sums cost ~log2(rows) bits of the per-slice difference (relative error
// ~1e-5 per view, well inside the 1e-4 bar, tests/test_gpu_parity.py).
//
// Footprint setup is lane-parallel (lane l sets up view vb + l, as in round
// 1): transverse trapezoid and column weights in fp32 (sf_common.cuh), axial
// map in f64 at the (sub-)voxel centre, stored relative to the table origin.
// Entries the table path cannot take (footprints wider than 4 columns, the
// second half of a split voxel, tables longer than B3_QMAX rows) take the
// direct per-row path.  No atomics: one lane owns each output voxel.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "sf_common.cuh"
#include "sf_launch.h"

#ifndef CTP_B3_WARPS
#define CTP_B3_WARPS 16  // a 1 x 16 strip of voxel columns along y per CTA (shared detector columns in L1)
#endif
// voxel columns of a CTA: 0: a 1 x B3_WARPS strip along y; TX > 0: a TX x
// (B3_WARPS / TX) tile (the footprints of nearby columns share detector
// columns: L1 reuse of the sinogram rows between the CTA's warps; measured:
// 2 x 8, 4 x 4, 8 x 2 within 1% of the strip on C3, 4 x 4 5% slower on C5)
#ifndef CTP_B3_TX
#define CTP_B3_TX 0
#endif
// L1 prefetch of the table rows (no registers, no scoreboard): 0: none, 1:
// every half of the view at the start of its table build (one L2 round trip
// per view instead of one per 128-row half), 2: the next view's halves
// before the current view's slices
#ifndef CTP_B3_PF
#define CTP_B3_PF 1
#endif
#ifndef CTP_B3_MINB
#define CTP_B3_MINB 2  // 64 registers: 32 resident warps per SM (measured best of 8/16 warps x 2-5 CTAs)
#endif
// rare paths (split halves, direct rows) inlined into the view loop: keeps the
// accumulators in place (no phi copies), at the cost of code size
#ifndef CTP_B3_INLINE_RARE
#define CTP_B3_INLINE_RARE 1
#endif
#if CTP_B3_INLINE_RARE
#define CTP_B3_RARE __forceinline__
#else
#define CTP_B3_RARE __noinline__
#endif

namespace ctp {

constexpr int B3_WARPS = CTP_B3_WARPS;  // warps per CTA: a 1 x B3_WARPS strip of voxel columns along y
constexpr int B3_NCF = 4;               // footprint columns of the table path

template <int ZPL>
struct B3Cfg {
  static constexpr int ZC = 32 * ZPL;  // slices per warp (lanes own lane + 32 m)
  // table rows: slices of B <= 1.5 rows plus margins, in whole 128-row chunks
  static constexpr int QMAX = ((ZC * 3 / 2 + 8) + 127) / 128 * 128;
};

struct B3Entry {  // one (sub-)voxel footprint of the warp's column in one view
  float W0;       // lower boundary of slice izs + 0.5, relative to the table origin R0
  float B;        // rows per slice
  float A;        // centre of slice izs relative to R0 (direct path)
  float lxy;
  float a0, a1;   // amp(i) = lxy sqrt(1 + (a0 + a1 i)^2), i = iz - izs
  int cl, ncol;   // footprint columns cl .. cl + ncol - 1 (ncol 0: no contribution)
  float ts[B3_NCF];
  int R0;         // table origin: absolute row, multiple of 4
  int n4;         // table rows / 4 (0: direct path)
  int mask;       // sub-footprints of this view (bit 1: second half of a split voxel)
  int pad;       // table base - 1 - 2^23 entries (shared address; see b3_eval)
};
static_assert(sizeof(B3Entry) == 64, "B3Entry layout");

template <int ZPL>
struct B3Smem {
  B3Entry ents[B3_WARPS][32];
  B3Entry split[B3_WARPS];
  // [4 + k]: I_k = sum_{j<=k} Q_j of table row k; [3] = 0 (k = -1)
  float tab[B3_WARPS][B3Cfg<ZPL>::QMAX + 4];
};

// Footprint of one (sub-)voxel for slices izs..ize: f64 axial map at the
// centre cxy, table origin and length, fp32 column weights.
template <int ZPL>
__device__ __forceinline__ void b3_fill(B3Entry& e, const SubFoot& f, const GridParams& gp, int izs, int ize,
                                        const ViewAx& ax, float2 cxy) {
  e.lxy = f.lxy;
  e.a1 = f.a1;
  e.a0 = fma_(f.a1, (float)izs, f.a0);
  e.cl = f.cl;
  e.ncol = f.ch >= f.cl ? f.ch - f.cl + 1 : 0;
  const Trap p = make_trap(f);
  float ts[B3_NCF];
  col_weights<B3_NCF>(p, f.cl, ts);
#pragma unroll
  for (int k = 0; k < B3_NCF; ++k) e.ts[k] = k < e.ncol ? ts[k] : 0.0f;
  double A, B;
  axial64(ax, gp.kind, (double)cxy.x, (double)cxy.y, A, B);
  const double Ts = fma(B, (double)izs, A), Te = fma(B, (double)ize, A);
  const double lo = Ts - 0.5 * B, hi = Te + 0.5 * B;
  // rows touched: row r spans [r - .5, r + .5)
  const double fa = floor(lo + 0.5), fz = floor(hi + 0.5);
  if (fz < 0.0 || fa > (double)(gp.nr - 1)) {  // entirely off the detector
    e.ncol = 0;
    e.n4 = 0;
    e.R0 = 0;
    e.W0 = e.B = e.A = 0.0f;
    return;
  }
  const int Ra = (int)fmax(fa, -1.0e6), Rz = (int)fmin(fz, 1.0e6);
  // origin one row below the first touched row (every boundary w >= 1, far
  // from the k = -1 edge under fp32 rounding), table one row past the last
  const int R0 = (Ra - 1) & ~3;
  const int n4 = (Rz - R0 + 2 + 3) >> 2;
  e.R0 = R0;
  e.W0 = (float)(lo + 0.5 - (double)R0);
  e.B = (float)B;
  e.A = (float)(Ts - (double)R0);
  const bool fast = e.ncol >= 1 && e.ncol <= B3_NCF && 4 * n4 <= B3Cfg<ZPL>::QMAX;
  e.n4 = fast ? n4 : 0;
}

// Lane-parallel setup of views vb + lane; the first sub-footprint goes to *e
// (the second half of a split voxel is rebuilt in the view loop).  Returns
// whether any view of the 32 splits the voxel.  Out of line: its registers
// stay out of the view loop's allocation.
template <int ZPL>
__device__ __noinline__ bool b3_setup(const GridParams& gp, const ViewCoef* __restrict__ vcoef,
                                      const ViewAx* __restrict__ vax, int vb, int ix, int iy, int izs, int ize,
                                      B3Entry* e, unsigned tab_adj) {
  const int v = vb + (threadIdx.x & 31);
  B3Entry E;
  E.ncol = 0;
  E.n4 = 0;
  E.R0 = 0;
  int mask = 0;
  if (v < gp.nv) {
    const ViewCoef vc = vcoef[v];
    SubFoot f0, f1;
    float2 c0, c1;
    mask = column_subs(vc, gp, ix, iy, f0, f1, c0, c1) & 3;
    if (mask & 1) b3_fill<ZPL>(E, f0, gp, izs, ize, vax[v], c0);
  }
  E.mask = mask;
  E.pad = (int)tab_adj;
  *e = E;
  return __any_sync(0xffffffffu, (mask & 2) != 0);
}

// Second half of a split voxel (_sf_subdivide, _kernels.py:542-552), rebuilt
// by one lane when a view needs it.
template <int ZPL>
__device__ CTP_B3_RARE void b3_split(const GridParams& gp, const ViewCoef* __restrict__ vcoef,
                                      const ViewAx* __restrict__ vax, int v, int ix, int iy, int izs, int ize,
                                      B3Entry* e, unsigned tab_adj) {
  SubFoot f0, f1;
  float2 c0, c1;
  const int mask = column_subs(vcoef[v], gp, ix, iy, f0, f1, c0, c1);
  B3Entry E;
  E.ncol = 0;
  E.n4 = 0;
  E.R0 = 0;
  E.mask = 0;
  if (mask & 2) b3_fill<ZPL>(E, f1, gp, izs, ize, vax[v], c1);
  E.pad = (int)tab_adj;
  *e = E;
}

// ---- table: I_k = sum_{j<=k} Q_j (+ a constant) of rows R0 + k, k < 4 n4 ---
// Q(r) = sum_c ts(c) y_c(r).  The input holds, per detector column, inclusive
// prefix sums P_c over aligned kBackSeg-row segments (sino_prefix.cu), so
// I(r) = B(seg(r)) + J(r), J = sum_c ts(c) P_c, with a base per segment:
// B(s + 1) = B(s) + J(last row of s), B(first) = 0 (the rows of the first
// segment before R0 add a constant, which the differences H(w') - H(w) drop).
// Lane t takes rows 128 h + 4 t .. + 3 of table half h; with R0 a multiple
// of 4 every half holds the same split: lanes t < o / 4 in one segment, the
// rest in the next (o = 128 - R0 mod 128, or 128: no split).  One shuffle per
// half (the first part's last row), no scans.
template <int NC, bool VEC, int QMAX>
__device__ __forceinline__ void b3_table_generic(float* __restrict__ tab, const float* __restrict__ yc, int nr,
                                                 int R0, int n4, const float* ts, int lane) {
  float carry = 0.0f;
  const int o4 = (((-R0) & (kBackSeg - 1)) ? ((-R0) & (kBackSeg - 1)) : kBackSeg) >> 2;
  const int nh = (4 * n4 + 127) >> 7;
#pragma unroll 1
  for (int h = 0; h < nh; ++h) {
    const int k0 = 128 * h + 4 * lane;  // table index of the lane's first row
    const int r0 = R0 + k0;
    float q[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    if (VEC) {
      // nr and R0 multiples of 4: a 4-row group is entirely on or off the
      // detector; a group past it in the last row's segment takes that row
      if (r0 >= 0 && r0 < nr) {
#pragma unroll
        for (int k = 0; k < NC; ++k) {
          const float4 a = __ldg(reinterpret_cast<const float4*>(yc + (size_t)k * nr + r0));
          q[0] = fmaf(ts[k], a.x, q[0]);
          q[1] = fmaf(ts[k], a.y, q[1]);
          q[2] = fmaf(ts[k], a.z, q[2]);
          q[3] = fmaf(ts[k], a.w, q[3]);
        }
      } else if (r0 >= nr && ((nr - 1) & ~(kBackSeg - 1)) == (r0 & ~(kBackSeg - 1))) {
        float v = 0.0f;
#pragma unroll
        for (int k = 0; k < NC; ++k) v = fmaf(ts[k], __ldg(yc + (size_t)k * nr + nr - 1), v);
        q[0] = q[1] = q[2] = q[3] = v;
      }
    } else {
      // rows before the detector read 0; rows past it keep the value of the
      // last on-detector row of their segment (0 in a segment past it)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int r = r0 + i, rc = min(r, nr - 1);
        if (r >= 0 && (rc & ~(kBackSeg - 1)) == (r & ~(kBackSeg - 1))) {
#pragma unroll
          for (int k = 0; k < NC; ++k) q[i] = fmaf(ts[k], __ldg(yc + (size_t)k * nr + rc), q[i]);
        }
      }
    }
    const float carry2 = carry + __shfl_sync(0xffffffffu, q[3], o4 - 1);
    const float base = lane < o4 ? carry : carry2;
    if (k0 < QMAX) reinterpret_cast<float4*>(tab)[k0 >> 2] = make_float4(base + q[0], base + q[1], base + q[2], base + q[3]);
    carry = carry2;
  }
}

// Fast table (every table row on the detector, 16-byte aligned): one 16-byte
// load per footprint column and half per lane (512 contiguous bytes per
// instruction), two packed FMAs, one shuffle per half.  (Issuing the loads of
// several halves ahead measured slower: more spills at 64 registers.)
__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// L1 prefetch of the rows b3_table_fast reads (nq rows of NC columns from yr)
template <int NC, int NCH>
__device__ __forceinline__ void b3_prefetch_rows(const float* __restrict__ yr, int nr, int nq, int lane) {
#pragma unroll
  for (int h = 0; h < 2 * NCH; ++h) {
    if (128 * h >= nq) break;  // warp-uniform
    if (128 * h + 4 * lane < nq) {
#pragma unroll
      for (int k = 0; k < NC; ++k) prefetch_l1(yr + k * nr + 128 * h + 4 * lane);
    }
  }
}

template <int NC, int NCH, int QMAX>
__device__ __forceinline__ void b3_table_fast(float* __restrict__ tab, const float* __restrict__ yc, int nr, int nq,
                                              int o4, const float* ts, int lane) {
  const float* p[NC];
  float2 T[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) {
    p[k] = yc + k * nr + 4 * lane;
    T[k] = bc2_(ts[k]);
  }
  float4* sp4 = reinterpret_cast<float4*>(tab + 4 * lane);
  float carry = 0.0f;
  const bool first = lane < o4;
  if (CTP_B3_PF == 1) b3_prefetch_rows<NC, NCH>(yc, nr, nq, lane);
#pragma unroll
  for (int h = 0; h < 2 * NCH; ++h) {
    if (128 * h >= nq) break;  // warp-uniform
    const bool ok = 128 * h + 4 * lane < nq;  // (rows past nq are never evaluated)
    float2 lo = make_float2(0.0f, 0.0f), hi = lo;
    if (ok) {
#pragma unroll
      for (int k = 0; k < NC; ++k) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(p[k] + 128 * h));
        lo = fma2_(T[k], make_float2(a.x, a.y), lo);
        hi = fma2_(T[k], make_float2(a.z, a.w), hi);
      }
    }
    // (lane o4 - 1's last row ends the first part's segment; when that lane
    // is past nq, no later row is evaluated)
    const float carry2 = carry + __shfl_sync(0xffffffffu, hi.y, o4 - 1);
    if (ok) {
      const float2 cc = bc2_(first ? carry : carry2);
      lo = add2_(lo, cc);
      hi = add2_(hi, cc);
      sp4[32 * h] = make_float4(lo.x, lo.y, hi.x, hi.y);
    }
    carry = carry2;
  }
}

template <int QMAX>
__device__ __forceinline__ float b3_eval(unsigned tab_adj, float w) {
  const float tf = __fadd_rd(w, 8388608.0f);
  const float fr = w - (tf - 8388608.0f);  // both subtractions exact
  const unsigned a = (unsigned)__float_as_int(tf) * 4u + tab_adj;  // one LEA
  // tab_adj points one entry below the table: (S0, S1) = (I_k-1, I_k), i.e.
  // H = S_k + fr Q_k with the exclusive S_k = I_k-1 and Q_k = I_k - I_k-1
  float S0, S1;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(S0) : "r"(a));
  asm volatile("ld.shared.f32 %0, [%1 + 4];" : "=f"(S1) : "r"(a));
  return fmaf(fr, S1 - S0, S0);
}

__device__ __forceinline__ float2 sub2_(float2 a, float2 b) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "sub.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
// (a + 2^23) rounded toward -inf, packed
__device__ __forceinline__ float2 add_rm_2p23_2_(float2 a) {
  float2 d;
  asm("{.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %4};\n\t"
      "add.rm.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;}"
      : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(8388608.0f));
  return d;
}

// Table lookups of a pair of boundaries (packed floor trick)
template <int QMAX>
__device__ __forceinline__ float2 b3_eval2(unsigned tab_adj, float2 w) {
  const float2 tf = add_rm_2p23_2_(w);
  const float2 fr = sub2_(w, add2_(tf, bc2_(-8388608.0f)));  // exact
  const unsigned a0 = (unsigned)__float_as_int(tf.x) * 4u + tab_adj;
  const unsigned a1 = (unsigned)__float_as_int(tf.y) * 4u + tab_adj;
  float S0, T0, S1, T1;  // (S_k, S_k+1) of both boundaries
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(S0) : "r"(a0));
  asm volatile("ld.shared.f32 %0, [%1 + 4];" : "=f"(T0) : "r"(a0));
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(S1) : "r"(a1));
  asm volatile("ld.shared.f32 %0, [%1 + 4];" : "=f"(T1) : "r"(a1));
  const float2 S = make_float2(S0, S1);
  return fma2_(fr, sub2_(make_float2(T0, T1), S), S);
}

// Slices lane + 32 m: x += amp (H(upper) - H(lower)); the lower boundary of
// slice lane + 32 m is the upper one of lane - 1 (lane 31 of step m - 1 for
// lane 0).  FULL: every lane has ZPL slices and every boundary lies in the
// table (steps evaluated in packed pairs); otherwise boundaries are clamped
// to the table and slices >= nvalid dropped.
template <int ZPL, bool FULL>
__device__ __forceinline__ void b3_slices(float2 (&acc)[ZPL / 2], const B3Entry& e, int lane, int nvalid) {
  constexpr int QMAX = B3Cfg<ZPL>::QMAX;
  const float W0 = e.W0, B = e.B;
  const float la1 = e.lxy * e.a1, la0 = e.lxy * e.a0, L2 = e.lxy * e.lxy;
  // S table base minus 2^23 entries, read from the entry (an opaque value:
  // the whole offset folds into one LEA per evaluation)
  const unsigned tab_adj = (unsigned)e.pad;
  const float wmax = (float)(4 * e.n4) - 0.5f;
  const float lf = (float)lane;
  // boundary w(i) = W0 + B i; this lane's upper boundaries i = lane + 1 + 32 m
  const float wl = fmaf(B, lf + 1.0f, W0), B32 = 32.0f * B;
  const float ql = fmaf(la1, lf, la0), la32 = 32.0f * la1;  // amp numerator at slice lane
  const int src = (lane + 31) & 31;
  if (FULL) {
    const float Hlo0 = b3_eval<QMAX>(tab_adj, fmaf(B, lf, W0));
    float rot_prev = 0.0f;
    static_assert(ZPL % 2 == 0, "pairs of steps");
#pragma unroll
    for (int m = 0; m < ZPL; m += 2) {
      const float2 w = make_float2(fmaf(B32, (float)m, wl), fmaf(B32, (float)(m + 1), wl));
      const float2 Hu = b3_eval2<QMAX>(tab_adj, w);
      const float r0 = __shfl_sync(0xffffffffu, Hu.x, src);
      const float r1 = __shfl_sync(0xffffffffu, Hu.y, src);
      const float2 Hl = make_float2(m == 0 ? Hlo0 : (lane == 0 ? rot_prev : r0), lane == 0 ? r0 : r1);
      rot_prev = r1;
      const float2 q = make_float2(fmaf(la32, (float)m, ql), fmaf(la32, (float)(m + 1), ql));
      const float2 t = fma2_(q, q, bc2_(L2));
      const float2 amp = make_float2(sqrt_approx(t.x), sqrt_approx(t.y));
      acc[m / 2] = fma2_(amp, sub2_(Hu, Hl), acc[m / 2]);
    }
    return;
  }
  auto H = [&](float w) { return b3_eval<QMAX>(tab_adj, fminf(fmaxf(w, 0.0f), wmax)); };
  const float Hlo0 = H(fmaf(B, lf, W0));
  float rot_prev = 0.0f;
#pragma unroll
  for (int m = 0; m < ZPL; ++m) {
    const float Hu = H(fmaf(B32, (float)m, wl));
    const float rot = __shfl_sync(0xffffffffu, Hu, src);
    const float Hl = m == 0 ? Hlo0 : (lane == 0 ? rot_prev : rot);
    rot_prev = rot;
    const float qa = fmaf(la32, (float)m, ql);
    const float amp = sqrt_approx(fmaf(qa, qa, L2));
    float& am = (m & 1) ? acc[m / 2].y : acc[m / 2].x;
    if (m < nvalid) am = fmaf(amp, Hu - Hl, am);
  }
}

// y_c(r) from the segment prefix sums of column c (sino_prefix.cu)
__device__ __forceinline__ float b3_row(const float* __restrict__ col, int r) {
  const float v = __ldg(col + r);
  return (r & (kBackSeg - 1)) ? v - __ldg(col + r - 1) : v;
}

// Direct path (wide footprints, split halves, long tables): rows r0 .. r0+K-1
// of one slice, any footprint width, rows off the detector skipped.
__device__ CTP_B3_RARE float b3_voxel_direct(float acc, float amp, float lo, float hi, const B3Entry& e,
                                              const Trap& wide, int K, const float* __restrict__ yv, int nr,
                                              int origin) {
  const float fl = row_floor(lo);  // r0 - 1 (rows relative to origin)
  const int r0 = (int)fl + 1 + origin;
  float g = clampf_(add_(fl, 0.5f), lo, hi);
  for (int k = 0; k < K; ++k) {
    const int r = r0 + k;
    const float gn = clampf_(add_(fl, (float)k + 1.5f), lo, hi);
    float q = 0.0f;
    if (r >= 0 && r < nr) {
      if (e.ncol <= B3_NCF) {
        for (int c = 0; c < e.ncol; ++c) q = fma_(e.ts[c], b3_row(yv + (size_t)(e.cl + c) * nr, r), q);
      } else {
        float prev = trap_cum(wide, sub_((float)e.cl, 0.5f));
        for (int c = 0; c < e.ncol; ++c) {
          const float cur = trap_cum(wide, add_((float)(e.cl + c), 0.5f));
          q = fma_(sub_(cur, prev), b3_row(yv + (size_t)(e.cl + c) * nr, r), q);
          prev = cur;
        }
      }
    }
    acc = fma_(mul_(amp, sub_(gn, g)), q, acc);
    g = gn;
  }
  return acc;
}

template <int ZPL, bool VEC, bool FULL>
__global__ void __launch_bounds__(B3_WARPS * 32, CTP_B3_MINB) sf_back3d_kernel(
    const __grid_constant__ GridParams gp, const ViewCoef* __restrict__ vcoef, const ViewAx* __restrict__ vax,
    const float* __restrict__ yT, float* __restrict__ out, int accumulate, int z0, int z1) {
  using Cfg = B3Cfg<ZPL>;
  extern __shared__ __align__(16) unsigned char b3_smem_raw[];
  B3Smem<ZPL>& SM = *reinterpret_cast<B3Smem<ZPL>*>(b3_smem_raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#if CTP_B3_TX
  constexpr int TY = B3_WARPS / CTP_B3_TX;
  const int ntx = (gp.nx + CTP_B3_TX - 1) / CTP_B3_TX;
  const int ix = (blockIdx.x % ntx) * CTP_B3_TX + warp % CTP_B3_TX;
  const int iy = (blockIdx.x / ntx) * TY + warp / CTP_B3_TX;
  if (ix >= gp.nx) return;
#else
  const int ix = blockIdx.x % gp.nx;
  const int iy = (blockIdx.x / gp.nx) * B3_WARPS + warp;
#endif
  if (iy >= gp.ny) return;  // warp-uniform; no CTA barriers below
  const int b = blockIdx.z;
  const int izs = z0 + blockIdx.y * Cfg::ZC;  // slices [z0, z1) of this launch
  const int ize = min(izs + Cfg::ZC, z1) - 1;
  const int nr = gp.nr;
  const size_t view_elems = (size_t)gp.nc * nr;
  const float* yb = yT + (size_t)b * gp.nv * view_elems;
  float* tab = SM.tab[warp] + 4;  // row k at tab[k]; tab[-1] = 0
  if (lane < 4) SM.tab[warp][lane] = 0.0f;
  // table base minus one entry minus 2^23 entries (b3_eval indexes it with
  // the float bits and reads (I_k-1, I_k))
  const unsigned tab_adj = (unsigned)__cvta_generic_to_shared(tab) - 4u - 0x4B000000u * 4u;
  B3Entry(&my)[32] = SM.ents[warp];
  B3Entry& sp = SM.split[warp];
  const int span = ize - izs;  // this lane's slices: izs + lane + 32 m, m < nvalid
  const int nvalid = lane > span ? 0 : min(ZPL, (span - lane) / 32 + 1);
  float2 acc[ZPL / 2];  // slices lane + 32 m: acc[m / 2].x (m even) / .y (m odd)
#pragma unroll
  for (int m = 0; m < ZPL / 2; ++m) acc[m] = make_float2(0.0f, 0.0f);

  for (int vb = 0; vb < gp.nv; vb += 32) {
    const bool split = b3_setup<ZPL>(gp, vcoef, vax, vb, ix, iy, izs, ize, &my[lane], tab_adj);
    __syncwarp();
    const int nvb = min(32, gp.nv - vb);
    // the direct (per-row) path: wide footprints, long tables, split halves
    auto direct = [&](const B3Entry& e, const float* yview, int v, bool second) {
      Trap wide{};
      if (e.ncol > B3_NCF) {  // rare: rebuild the breakpoints of this footprint
        SubFoot f0, f1;
        column_footprint(vcoef[v], gp, ix, iy, f0, f1);
        wide = make_trap(second ? f1 : f0);
      }
      const int K = rows_per_slice(e.B);
      const float E = 0.5f * e.B;
#pragma unroll
      for (int m = 0; m < ZPL; ++m) {  // (unrolled: acc stays in registers)
        if (m >= nvalid) break;
        const float izf = (float)(lane + 32 * m);
        const float T = fma_(e.B, izf, e.A);
        const float lo = sub_(T, E), hi = add_(T, E);
        const float q = fma_(e.a1, izf, e.a0);
        const float amp = mul_(e.lxy, sqrt_approx(fma_(q, q, 1.0f)));
        float& am = (m & 1) ? acc[m / 2].y : acc[m / 2].x;
        am = b3_voxel_direct(am, amp, lo, hi, e, wide, K, yview, nr, e.R0);
      }
    };
    const float* yview = yb + (size_t)vb * view_elems;  // [c][r] of view vb + j
    for (int j = 0; j < nvb; ++j, yview += view_elems) {
      const B3Entry& e = my[j];
      const int ncol = e.ncol;
      if (ncol > 0 && e.n4 > 0) {
        const float* yc = yview + (size_t)e.cl * nr;
        const float* ts = e.ts;  // (read from the shared entry: no local copy)
        constexpr int NCH = (Cfg::QMAX + 255) / 256;
        if (VEC && e.R0 >= 0 && e.R0 + 4 * e.n4 <= nr) {
          const float* yr = yc + e.R0;
          const int nq = 4 * e.n4;
          // lanes of each half before the segment boundary (all: none inside)
          const int o4 = (((-e.R0) & (kBackSeg - 1)) ? ((-e.R0) & (kBackSeg - 1)) : kBackSeg) >> 2;
          switch (ncol) {  // warp-uniform: load only the footprint's columns
            case 1: b3_table_fast<1, NCH, Cfg::QMAX>(tab, yr, nr, nq, o4, ts, lane); break;
            case 2: b3_table_fast<2, NCH, Cfg::QMAX>(tab, yr, nr, nq, o4, ts, lane); break;
            case 3: b3_table_fast<3, NCH, Cfg::QMAX>(tab, yr, nr, nq, o4, ts, lane); break;
            default: b3_table_fast<4, NCH, Cfg::QMAX>(tab, yr, nr, nq, o4, ts, lane); break;
          }
        } else {
          switch (ncol) {
            case 1: b3_table_generic<1, VEC, Cfg::QMAX>(tab, yc, nr, e.R0, e.n4, ts, lane); break;
            case 2: b3_table_generic<2, VEC, Cfg::QMAX>(tab, yc, nr, e.R0, e.n4, ts, lane); break;
            case 3: b3_table_generic<3, VEC, Cfg::QMAX>(tab, yc, nr, e.R0, e.n4, ts, lane); break;
            default: b3_table_generic<4, VEC, Cfg::QMAX>(tab, yc, nr, e.R0, e.n4, ts, lane); break;
          }
        }
        __syncwarp();
        if (CTP_B3_PF == 2 && j + 1 < nvb) {  // the next view's rows into L1
          const B3Entry& en = my[j + 1];
          if (en.ncol > 0 && en.n4 > 0 && en.R0 >= 0 && en.R0 + 4 * en.n4 <= nr) {
            constexpr int NCH = (Cfg::QMAX + 255) / 256;
            const float* yr = yview + view_elems + (size_t)en.cl * nr + en.R0;
            switch (en.ncol) {
              case 1: b3_prefetch_rows<1, NCH>(yr, nr, 4 * en.n4, lane); break;
              case 2: b3_prefetch_rows<2, NCH>(yr, nr, 4 * en.n4, lane); break;
              case 3: b3_prefetch_rows<3, NCH>(yr, nr, 4 * en.n4, lane); break;
              default: b3_prefetch_rows<4, NCH>(yr, nr, 4 * en.n4, lane); break;
            }
          }
        }
        b3_slices<ZPL, FULL>(acc, e, lane, nvalid);
        __syncwarp();
      } else if (ncol > 0) {
        direct(e, yview, vb + j, false);
      }
      if (split && (e.mask & 2)) {  // second half of a split voxel (rare): rebuilt, direct path
        __syncwarp();  // every lane is done with the previous split entry
        if (lane == 0) b3_split<ZPL>(gp, vcoef, vax, vb + j, ix, iy, izs, ize, &sp, tab_adj);
        __syncwarp();
        if (sp.ncol > 0) direct(sp, yview, vb + j, true);
      }
    }
    __syncwarp();
  }
  // out[b][iz][iy][ix]
  const size_t plane = (size_t)gp.ny * gp.nx;
  float* ob = out + (size_t)b * plane * gp.nz + (size_t)iy * gp.nx + ix;
#pragma unroll
  for (int m = 0; m < ZPL; ++m) {
    if (m >= nvalid) break;
    float* p = ob + (size_t)(izs + lane + 32 * m) * plane;
    const float am = (m & 1) ? acc[m / 2].y : acc[m / 2].x;
    *p = accumulate ? (*p + am) : am;
  }
}

// FULL z-blocks (every lane has ZPL slices) and the partial last one are
// separate instantiations, so the full blocks' slice loop has no clamps.
template <int ZPL, bool VEC, bool FULL>
static cudaError_t launch_back3d_t(const GridParams& gp, const ViewCoef* vcoef, const ViewAx* vax,
                                   const float* yT, float* vol, int batch, bool accumulate, cudaStream_t st,
                                   int z0, int z1) {
  auto kern = sf_back3d_kernel<ZPL, VEC, FULL>;
  const int smem = (int)sizeof(B3Smem<ZPL>);
  cudaError_t ea = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (ea != cudaSuccess) return ea;
#if CTP_B3_TX
  const int nbx = (gp.nx + CTP_B3_TX - 1) / CTP_B3_TX;
  const int nby = (gp.ny + B3_WARPS / CTP_B3_TX - 1) / (B3_WARPS / CTP_B3_TX);
#else
  const int nbx = gp.nx;
  const int nby = (gp.ny + B3_WARPS - 1) / B3_WARPS;
#endif
  const size_t sino_elems = (size_t)gp.nv * gp.nr * gp.nc;
  const size_t vol_elems = (size_t)gp.nx * gp.ny * gp.nz;
  for (int b0 = 0; b0 < batch; b0 += 65535) {
    const int nb = min(65535, batch - b0);
    const dim3 grid(nbx * nby, (z1 - z0 + B3Cfg<ZPL>::ZC - 1) / B3Cfg<ZPL>::ZC, nb);
    kern<<<grid, B3_WARPS * 32, smem, st>>>(gp, vcoef, vax, yT + (size_t)b0 * sino_elems,
                                            vol + (size_t)b0 * vol_elems, accumulate ? 1 : 0, z0, z1);
  }
  return cudaGetLastError();
}

template <int ZPL, bool VEC>
static cudaError_t launch_back3d_z(const GridParams& gp, const ViewCoef* vcoef, const ViewAx* vax,
                                   const float* yT, float* vol, int batch, bool accumulate, cudaStream_t st,
                                   int z0, int z1) {
  constexpr int ZC = B3Cfg<ZPL>::ZC;
  const int zf = z0 + (z1 - z0) / ZC * ZC;  // end of the full z-blocks
  cudaError_t e = cudaSuccess;
  if (zf > z0) e = launch_back3d_t<ZPL, VEC, true>(gp, vcoef, vax, yT, vol, batch, accumulate, st, z0, zf);
  if (e == cudaSuccess && z1 > zf)
    e = launch_back3d_t<ZPL, VEC, false>(gp, vcoef, vax, yT, vol, batch, accumulate, st, zf, z1);
  return e;
}

cudaError_t launch_back(const GridParams& gp, const ViewCoef* vcoef, const ViewAx* vax, const float* yT,
                        float* vol, int batch, bool accumulate, cudaStream_t st, int z0, int z1) {
  if (z1 < 0) z1 = gp.nz;
  if (z0 < 0 || z0 >= z1 || z1 > gp.nz) return cudaErrorInvalidValue;
  if (back_legacy()) return launch_back_legacy(  // A/B against round 1's kernel (raw input)
      gp, vcoef, vax, yT, vol, batch, accumulate, st, z0, z1);
  const bool vec = gp.nr % 4 == 0 && (reinterpret_cast<uintptr_t>(yT) & 15) == 0;
  static const int zpl_env = getenv("CTP_B3_ZPL") ? atoi(getenv("CTP_B3_ZPL")) : 16;  // (tuning)
  // slices per warp: 512 (16 per lane) for tall z-ranges, 256 for the
  // 256-slice z-chunks of the sharded back projection (dist.cu), else 128
  if ((zpl_env == 8 || z1 - z0 < 384) && z1 - z0 >= 192)
    return vec ? launch_back3d_z<8, true>(gp, vcoef, vax, yT, vol, batch, accumulate, st, z0, z1)
               : launch_back3d_z<8, false>(gp, vcoef, vax, yT, vol, batch, accumulate, st, z0, z1);
  if (z1 - z0 >= 384)
    return vec ? launch_back3d_z<16, true>(gp, vcoef, vax, yT, vol, batch, accumulate, st, z0, z1)
               : launch_back3d_z<16, false>(gp, vcoef, vax, yT, vol, batch, accumulate, st, z0, z1);
  return vec ? launch_back3d_z<4, true>(gp, vcoef, vax, yT, vol, batch, accumulate, st, z0, z1)
             : launch_back3d_z<4, false>(gp, vcoef, vax, yT, vol, batch, accumulate, st, z0, z1);
}

}  // namespace ctp
