// sf_kernels.cu -- sm_100a kernels of the SF-TR projector pair.
//
//   sf_forward_kernel : y = A x,  ray-driven GATHER.  One CTA owns a detector
//                       tile (view v, FW_CW columns, FW_ROWS rows) and gathers
//                       every voxel column whose footprint reaches the tile
//                       (reference: voxel-driven scatter into an f64 scratch
//                       per view, _kernels.py:555-663).
//   sf_back_kernel    : x = A^T y, voxel-driven GATHER.  One warp owns one
//                       voxel column x BK_ZC slices, lanes along z, and loops
//                       over all views (reference: _kernels.py:666-763).
//   transpose_kernel  : [batch][R][C] -> [batch][C][R] layout change used to
//                       make the z (volume) / row (sinogram) axis contiguous.
//
// No atomics anywhere; every output element is produced by exactly one
// thread with a fixed summation order, so results are deterministic.
// Both kernels take the footprint coefficients from sf_common.cuh so that the
// pair is an exact fp32 transpose (see that header).
#include <cuda_runtime.h>

#include <cstdint>

#include "sf_common.cuh"
#include "sf_launch.h"

namespace ctp {

// ---------------------------------------------------------------------------
// layout transpose
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) transpose_kernel(const float* __restrict__ in,
                                                        float* __restrict__ out, int R, int C,
                                                        int batch0) {
  __shared__ float tile[32][33];
  const int b = blockIdx.z + batch0;
  const size_t off = (size_t)b * (size_t)R * (size_t)C;
  const int c_base = blockIdx.x * 32, r_base = blockIdx.y * 32;
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
constexpr int BK_WARPS = 8;
constexpr int BK_ZPL = 4;              // voxels per lane
constexpr int BK_ZC = 32 * BK_ZPL;     // slices per warp
constexpr int BK_QBUF = 640;           // per-warp Q staging (rows)
constexpr int BK_MAXC = 8;             // footprint columns kept in registers

// Q(r) = sum_c ts(c) * y[v][c][r]  (column sum first; fixed ascending-c order)
__device__ __forceinline__ float q_value(const SubFoot& f, const float (&ts)[BK_MAXC], int ncols,
                                         const float* __restrict__ yv, int nr, int r) {
  float q = 0.0f;
  if (ncols <= BK_MAXC) {
#pragma unroll
    for (int k = 0; k < BK_MAXC; ++k)
      if (k < ncols) q = fma_(ts[k], __ldg(yv + (size_t)(f.cl + k) * nr + r), q);
  } else {
    for (int c = f.cl; c <= f.ch; ++c) q = fma_(col_weight(f, c), __ldg(yv + (size_t)c * nr + r), q);
  }
  return q;
}

__device__ __forceinline__ void back_sub(const SubFoot& f, const GridParams& gp,
                                         const float* __restrict__ yv, float* qw, int lane,
                                         int izs, int ize, float (&acc)[BK_ZPL]) {
  if (f.cl > f.ch) return;
  const int nr = gp.nr;
  int Ra = (int)floorf(sub_(sub_(row_center(f, izs), f.E), 0.5f));
  int Rb = (int)ceilf(add_(add_(row_center(f, ize), f.E), 0.5f));
  Ra = Ra < 0 ? 0 : Ra;
  Rb = Rb > nr - 1 ? nr - 1 : Rb;
  if (Ra > Rb) return;
  const int nq = Rb - Ra + 1;
  const int ncols = f.ch - f.cl + 1;
  float ts[BK_MAXC];
#pragma unroll
  for (int k = 0; k < BK_MAXC; ++k) ts[k] = (k < ncols) ? col_weight(f, f.cl + k) : 0.0f;
  const bool table = nq <= BK_QBUF;
  if (table) {
    for (int j = lane; j < nq; j += 32) qw[j] = q_value(f, ts, ncols, yv, nr, Ra + j);
    __syncwarp();
  }
#pragma unroll
  for (int m = 0; m < BK_ZPL; ++m) {
    const int iz = izs + lane + 32 * m;
    if (iz > ize) continue;
    const float T = row_center(f, iz);
    const float lo = sub_(T, f.E), hi = add_(T, f.E);
    const float amp = amplitude(f, iz);
    int r0 = (int)floorf(sub_(lo, 0.5f));
    int r1 = (int)ceilf(add_(hi, 0.5f));
    r0 = r0 < Ra ? Ra : r0;
    r1 = r1 > Rb ? Rb : r1;
    float a = acc[m];
    for (int r = r0; r <= r1; ++r) {
      const float tt = row_overlap(lo, hi, r);
      const float q = table ? qw[r - Ra] : q_value(f, ts, ncols, yv, nr, r);
      a = fma_(mul_(amp, tt), q, a);
    }
    acc[m] = a;
  }
  if (table) __syncwarp();
}

__global__ void __launch_bounds__(BK_WARPS * 32) sf_back_kernel(GridParams gp,
                                                                const ViewCoef* __restrict__ vcoef,
                                                                const float* __restrict__ yT,
                                                                float* __restrict__ out,
                                                                int accumulate) {
  __shared__ float qbuf[BK_WARPS][BK_QBUF];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nbx = (gp.nx + 3) >> 2;
  const int ix = (blockIdx.x % nbx) * 4 + (warp & 3);
  const int iy = (blockIdx.x / nbx) * 2 + (warp >> 2);
  if (ix >= gp.nx || iy >= gp.ny) return;  // warp-uniform; no CTA barriers below
  const int b = blockIdx.z;
  const int izs = blockIdx.y * BK_ZC;
  const int ize = min(izs + BK_ZC, gp.nz) - 1;
  const size_t sino_elems = (size_t)gp.nv * gp.nr * gp.nc;
  const float* yb = yT + (size_t)b * sino_elems;
  float* qw = qbuf[warp];
  float acc[BK_ZPL];
#pragma unroll
  for (int m = 0; m < BK_ZPL; ++m) acc[m] = 0.0f;

  for (int v = 0; v < gp.nv; ++v) {
    const ViewCoef vc = vcoef[v];
    SubFoot f0, f1;
    const int mask = column_footprint(vc, gp, ix, iy, f0, f1);
    if (mask == 0) continue;
    const float* yv = yb + (size_t)v * gp.nc * gp.nr;  // [c][r] of view v
    if (mask & 1) back_sub(f0, gp, yv, qw, lane, izs, ize, acc);
    if (mask & 2) back_sub(f1, gp, yv, qw, lane, izs, ize, acc);
  }
  // out[b][iz][iy][ix]
  const size_t plane = (size_t)gp.ny * gp.nx;
  float* ob = out + (size_t)b * plane * gp.nz + (size_t)iy * gp.nx + ix;
#pragma unroll
  for (int m = 0; m < BK_ZPL; ++m) {
    const int iz = izs + lane + 32 * m;
    if (iz > ize) continue;
    float* p = ob + (size_t)iz * plane;
    *p = accumulate ? (*p + acc[m]) : acc[m];
  }
}

// ---------------------------------------------------------------------------
// forward projection: y = A x
// ---------------------------------------------------------------------------
constexpr int FW_WARPS = 8;
constexpr int FW_THREADS = FW_WARPS * 32;
constexpr int FW_CW = 8;                      // detector columns per tile
constexpr int FW_KR = 3;                      // 32-row groups per warp
constexpr int FW_ROWS = FW_WARPS * 32 * FW_KR;  // rows per tile
constexpr int FW_BATCH = FW_THREADS;          // candidate columns per setup round
constexpr int FW_VBUF = 256;                  // per-warp amp*x staging (slices)

struct FwEntry {
  int col;        // iy*nx + ix
  float A, B, E;  // axial map
  float lxy, a0, a1;
  float invB;
  float ts[FW_CW];  // transverse weights of the tile's columns (0 outside [cl,ch])
};
static_assert(sizeof(FwEntry) == 64, "FwEntry layout");

size_t forward_smem_bytes(int n_primary) {
  return sizeof(FwEntry) * 2 * FW_BATCH + sizeof(float) * FW_WARPS * FW_VBUF +
         sizeof(int) * (2 * (size_t)n_primary + 2) + sizeof(int) * 2 * (FW_WARPS + 1);
}

__device__ __forceinline__ bool reaches_tile(const SubFoot& f, const GridParams& gp, int c0, int cw,
                                             float band_lo, float band_hi) {
  const bool cols_ok = max(f.cl, c0) <= min(f.ch, c0 + cw - 1);
  const float tlo = sub_(row_center(f, 0), f.E);
  const float thi = add_(row_center(f, gp.nz - 1), f.E);
  return cols_ok && thi > band_lo && tlo < band_hi;
}

__device__ __forceinline__ void write_entry(FwEntry& e, const SubFoot& f, int col, int c0, int cw) {
  e.col = col;
  e.A = f.A; e.B = f.B; e.E = f.E;
  e.lxy = f.lxy; e.a0 = f.a0; e.a1 = f.a1;
  e.invB = 1.0f / f.B;
#pragma unroll
  for (int c = 0; c < FW_CW; ++c) {
    const int cc = c0 + c;
    e.ts[c] = (c < cw && cc >= f.cl && cc <= f.ch) ? col_weight(f, cc) : 0.0f;
  }
}

// exclusive scan of one int per thread over the CTA; returns the total
__device__ __forceinline__ int block_exclusive_scan(int val, int* warp_tot, int& total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int inc = val;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const int n = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += n;
  }
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int w = 0; w < FW_WARPS; ++w) {
      const int t = warp_tot[w];
      warp_tot[w] = run;
      run += t;
    }
    warp_tot[FW_WARPS] = run;
  }
  __syncthreads();
  const int excl = warp_tot[warp] + inc - val;
  total = warp_tot[FW_WARPS];
  __syncthreads();
  return excl;
}

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
  const float k = s_mm / gp.hx;
  px = vc.xc0 + k * vc.ux;
  py = vc.yc0 + k * vc.uy;
  if (gp.kind == kParallel) {
    dx = vc.wx; dy = vc.wy;
  } else {
    dx = px - vc.xs; dy = py - vc.ys;
  }
}

__global__ void __launch_bounds__(FW_THREADS) sf_forward_kernel(GridParams gp,
                                                                const ViewCoef* __restrict__ vcoef,
                                                                const float* __restrict__ xT,
                                                                float* __restrict__ y,
                                                                int accumulate, int view_batch0) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  FwEntry* ent = reinterpret_cast<FwEntry*>(smem_raw);
  float* xabuf = reinterpret_cast<float*>(ent + 2 * FW_BATCH);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  const int vb = blockIdx.z + view_batch0;
  const int v = vb % gp.nv, b = vb / gp.nv;
  const int c0 = blockIdx.x * FW_CW;
  const int cw = min(FW_CW, gp.nc - c0);
  const int R0 = blockIdx.y * FW_ROWS;
  const ViewCoef vc = vcoef[v];

  // ---- 1. strip of candidate voxel columns (wedge between the tile's edge rays)
  float plx, ply, dlx, dly, phx, phy, dhx, dhy;
  edge_ray(vc, gp, (float)c0 - 0.5f, plx, ply, dlx, dly);
  edge_ray(vc, gp, (float)(c0 + cw) - 0.5f, phx, phy, dhx, dhy);
  const float nl = rsqrtf(dlx * dlx + dly * dly), nh = rsqrtf(dhx * dhx + dhy * dhy);
  const bool primary_x = fabsf(dlx) * nl + fabsf(dhx) * nh >= fabsf(dly) * nl + fabsf(dhy) * nh;
  const int nP = primary_x ? gp.nx : gp.ny, nQ = primary_x ? gp.ny : gp.nx;
  const float halfP = primary_x ? gp.half_x : gp.half_y, halfQ = primary_x ? gp.half_y : gp.half_x;
  // rays as (p, q) = (primary, secondary) components
  const float lp = primary_x ? plx : ply, lq = primary_x ? ply : plx;
  const float ldp = primary_x ? dlx : dly, ldq = primary_x ? dly : dlx;
  const float hp = primary_x ? phx : phy, hq = primary_x ? phy : phx;
  const float hdp = primary_x ? dhx : dhy, hdq = primary_x ? dhy : dhx;
  const bool cull = vc.cull && fabsf(ldp) * nl > 1e-3f && fabsf(hdp) * nh > 1e-3f;
  const float lslope = cull ? ldq / ldp : 0.0f, hslope = cull ? hdq / hdp : 0.0f;

  int* prefix = reinterpret_cast<int*>(xabuf + FW_WARPS * FW_VBUF);  // nP + 1
  int* jlo = prefix + (nP + 1);                                      // nP
  int* scan_tmp = jlo + nP + 1;                                      // FW_WARPS + 1
  const int seg = (nP + FW_THREADS - 1) / FW_THREADS;
  int my_sum = 0;
  for (int t = 0; t < seg; ++t) {
    const int i = tid * seg + t;
    if (i >= nP) break;
    int jl = 0, jh = nQ - 1;
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
    const int n = jh >= jl ? jh - jl + 1 : 0;
    jlo[i] = jl;
    prefix[i] = n;  // counts for now
    my_sum += n;
  }
  __syncthreads();
  int total;
  int run = block_exclusive_scan(my_sum, scan_tmp, total);
  for (int t = 0; t < seg; ++t) {
    const int i = tid * seg + t;
    if (i >= nP) break;
    const int n = prefix[i];
    prefix[i] = run;
    run += n;
  }
  if (tid == 0) prefix[nP] = total;
  __syncthreads();

  // ---- 2. accumulate the tile
  float acc[FW_KR][FW_CW];
#pragma unroll
  for (int k = 0; k < FW_KR; ++k)
#pragma unroll
    for (int c = 0; c < FW_CW; ++c) acc[k][c] = 0.0f;

  const int rw0 = R0 + warp * 32 * FW_KR;
  const int rw1 = min(rw0 + 32 * FW_KR, gp.nr) - 1;  // last row of this warp
  const float band_lo = (float)R0 - 0.5f;
  const float band_hi = (float)min(R0 + FW_ROWS, gp.nr) - 0.5f;
  const size_t ncolvox = (size_t)gp.nx * gp.ny;
  const float* xb = xT + (size_t)b * ncolvox * gp.nz;
  float* xw = xabuf + warp * FW_VBUF;

  for (int base = 0; base < total; base += FW_BATCH) {
    // 2a. one candidate per thread -> footprint setup -> compacted entries
    const int k = base + tid;
    SubFoot f0, f1;
    int mask = 0, col = 0;
    if (k < total) {
      int lo = 0, hi = nP;
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (prefix[mid] <= k) lo = mid; else hi = mid;
      }
      const int i = lo, j = jlo[i] + (k - prefix[i]);
      const int ix = primary_x ? i : j, iy = primary_x ? j : i;
      col = iy * gp.nx + ix;
      mask = column_footprint(vc, gp, ix, iy, f0, f1);
      // keep sub-footprints that reach the tile's columns and row band
      if ((mask & 1) && !reaches_tile(f0, gp, c0, cw, band_lo, band_hi)) mask &= ~1;
      if ((mask & 2) && !reaches_tile(f1, gp, c0, cw, band_lo, band_hi)) mask &= ~2;
    }
    const int cnt = __popc(mask);
    int nent;
    const int off = block_exclusive_scan(cnt, scan_tmp, nent);
    if (mask & 1) write_entry(ent[off], f0, col, c0, cw);
    if (mask & 2) write_entry(ent[off + (mask & 1)], f1, col, c0, cw);
    __syncthreads();

    // 2b. every warp gathers every entry into its own rows
    if (rw0 <= rw1) {
      for (int e = 0; e < nent; ++e) {
        const FwEntry& E = ent[e];
        SubFoot f;
        f.A = E.A; f.B = E.B; f.E = E.E; f.lxy = E.lxy; f.a0 = E.a0; f.a1 = E.a1;
        const float invB = E.invB;
        // slices whose axial interval can reach rows [rw0, rw1]
        int za = (int)floorf(((float)rw0 - 0.5f - f.E - f.A) * invB) - 1;
        int zb = (int)ceilf(((float)rw1 + 0.5f + f.E - f.A) * invB) + 1;
        za = max(za, 0);
        zb = min(zb, gp.nz - 1);
        if (za > zb) continue;
        const float* xc = xb + (size_t)E.col * gp.nz;
        float P[FW_KR];
#pragma unroll
        for (int kk = 0; kk < FW_KR; ++kk) P[kk] = 0.0f;
        for (int piece = za; piece <= zb; piece += FW_VBUF) {
          const int pe = min(piece + FW_VBUF - 1, zb);
          for (int iz = piece + lane; iz <= pe; iz += 32)
            xw[iz - piece] = mul_(amplitude(f, iz), __ldg(xc + iz));
          __syncwarp();
#pragma unroll
          for (int kk = 0; kk < FW_KR; ++kk) {
            const int r = rw0 + 32 * kk + lane;
            if (r > rw1) continue;
            int z0 = (int)floorf(((float)r - 0.5f - f.E - f.A) * invB) - 1;
            int z1 = (int)ceilf(((float)r + 0.5f + f.E - f.A) * invB) + 1;
            z0 = max(z0, piece);
            z1 = min(z1, pe);
            float p = P[kk];
            for (int iz = z0; iz <= z1; ++iz) {
              const float T = row_center(f, iz);
              const float tt = row_overlap(sub_(T, f.E), add_(T, f.E), r);
              p = fma_(tt, xw[iz - piece], p);
            }
            P[kk] = p;
          }
          __syncwarp();
        }
#pragma unroll
        for (int kk = 0; kk < FW_KR; ++kk)
#pragma unroll
          for (int c = 0; c < FW_CW; ++c) acc[kk][c] = fma_(E.ts[c], P[kk], acc[kk][c]);
      }
    }
    __syncthreads();  // entries are overwritten by the next round
  }

  // ---- 3. store the tile: y[b][v][r][c0 + c]
  float* yv = y + ((size_t)b * gp.nv + v) * (size_t)gp.nr * gp.nc;
#pragma unroll
  for (int kk = 0; kk < FW_KR; ++kk) {
    const int r = rw0 + 32 * kk + lane;
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
// launchers
// ---------------------------------------------------------------------------
cudaError_t launch_transpose(const float* in, float* out, int R, int C, int batch,
                             cudaStream_t st) {
  const dim3 block(256);
  for (int b0 = 0; b0 < batch; b0 += 65535) {
    const int nb = min(65535, batch - b0);
    const dim3 grid((C + 31) / 32, (R + 31) / 32, nb);
    transpose_kernel<<<grid, block, 0, st>>>(in, out, R, C, b0);
  }
  return cudaGetLastError();
}

cudaError_t launch_back(const GridParams& gp, const ViewCoef* vcoef, const float* yT, float* vol,
                        int batch, bool accumulate, cudaStream_t st) {
  const int nbx = (gp.nx + 3) / 4, nby = (gp.ny + 1) / 2;
  for (int b0 = 0; b0 < batch; b0 += 65535) {
    const int nb = min(65535, batch - b0);
    const dim3 grid(nbx * nby, (gp.nz + BK_ZC - 1) / BK_ZC, nb);
    const size_t sino_elems = (size_t)gp.nv * gp.nr * gp.nc;
    const size_t vol_elems = (size_t)gp.nx * gp.ny * gp.nz;
    sf_back_kernel<<<grid, BK_WARPS * 32, 0, st>>>(gp, vcoef, yT + (size_t)b0 * sino_elems,
                                                   vol + (size_t)b0 * vol_elems, accumulate ? 1 : 0);
  }
  return cudaGetLastError();
}

cudaError_t launch_forward(const GridParams& gp, const ViewCoef* vcoef, const float* xT, float* sino,
                           int batch, bool accumulate, cudaStream_t st) {
  const int nP = gp.nx > gp.ny ? gp.nx : gp.ny;
  const size_t smem = forward_smem_bytes(nP);
  cudaError_t e = cudaFuncSetAttribute(sf_forward_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int total = gp.nv * batch;
  for (int z0 = 0; z0 < total; z0 += 65535) {
    const int nz = min(65535, total - z0);
    const dim3 grid((gp.nc + FW_CW - 1) / FW_CW, (gp.nr + FW_ROWS - 1) / FW_ROWS, nz);
    sf_forward_kernel<<<grid, FW_THREADS, smem, st>>>(gp, vcoef, xT, sino, accumulate ? 1 : 0, z0);
  }
  return cudaGetLastError();
}

}  // namespace ctp
