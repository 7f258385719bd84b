/*
 * ctproj_b200.h -- C-ABI of the B200-native separable-footprint (SF-TR)
 * projector pair.  Plain pointers, sizes and POD structs only; no torch or
 * CUDA types appear in any signature (streams are passed as void*).
 *
 * Each entry point replaces one piece of the reference package `ctproj`
 * (a numba CPU implementation, /root/reference/pkg/src/ctproj):
 *
 *   ctp_geom                <- the 17-tuple built by kernel_geom()
 *                              (pkg/src/ctproj/_common.py:8-39) from
 *                              pose_table() (pkg/src/ctproj/geometry.py:227-263);
 *                              `back` is omitted, as sf.py:35/44 drops it.
 *   ctp_plan_create         <- the per-call kernel_geom()/pose_table() flattening,
 *                              hoisted out of the hot path: per-view footprint
 *                              coefficients are derived once (f64 on the host)
 *                              and kept resident on the device.
 *   ctp_sf_forward          <- sf_forward_kernel(vol, out, kind, src, c0, u, vax,
 *                              w, pw, ph, cr, cc, sdd, x0, y0, z0, hx, hz)
 *                              (pkg/src/ctproj/_kernels.py:650-663), called by
 *                              sf_forward (pkg/src/ctproj/sf.py:30-36) and, per
 *                              batch element, by operator.forward (operator.py:59-66).
 *   ctp_sf_back             <- sf_back_kernel(y, out, ...same...)
 *                              (pkg/src/ctproj/_kernels.py:666-763), called by
 *                              sf_backproject (sf.py:39-45) / operator.adjoint
 *                              (operator.py:69-75).
 *   ctp_sf_forward_oneshot  <- the exact reference kernel shape: geometry in,
 *   ctp_sf_back_oneshot        arrays in/out, no persistent state.
 *
 * Contract (mirrors the reference kernels):
 *   - the caller allocates the output; it is fully overwritten (never read)
 *     unless CTP_FLAG_ACCUMULATE is passed;
 *   - inputs are read-only and must not alias the output;
 *   - volumes are f32 [batch][nz][ny][nx], sinograms f32 [batch][nv][nr][nc],
 *     C-contiguous, in DEVICE memory;
 *   - calls are stream-ordered and never synchronise the host;
 *   - validation happens before launch and is reported by status code; the
 *     kernels themselves never fail (degenerate geometry contributes 0, as the
 *     reference's ok=False paths do, _kernels.py:468-469, 475-476, 511-520);
 *   - results are deterministic: no atomics, fixed reduction order.
 */
#ifndef CTPROJ_B200_H
#define CTPROJ_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CTP_ABI_VERSION 2

/* geometry kinds; same codes as KIND_CODE (pkg/src/ctproj/_common.py:5) */
enum ctp_kind {
  CTP_PARALLEL = 0,
  CTP_CONE_FLAT = 1,
  CTP_CONE_CURVED = 2,
  CTP_MODULAR = 3
};

/* status codes; the Python layer maps them onto the reference exception
 * classes (pkg/src/ctproj/errors.py) */
enum ctp_status {
  CTP_OK = 0,
  CTP_ERR_INVALID_ARGUMENT = 1,     /* -> InvalidValueError / ValueError */
  CTP_ERR_UNSUPPORTED_GEOMETRY = 2, /* -> UnsupportedGeometryError (sf.py:23-27) */
  CTP_ERR_SPEC_MISMATCH = 3,        /* -> SpecMismatchError */
  CTP_ERR_CUDA = 4,                 /* CUDA runtime failure (message via ctp_last_error) */
  CTP_ERR_OUT_OF_MEMORY = 5,
  CTP_ERR_WORKSPACE = 6             /* workspace too small */
};

/* flags for ctp_sf_forward / ctp_sf_back */
#define CTP_FLAG_ACCUMULATE 1u /* out += A x (resp. A^T y) instead of out = ... */
#define CTP_FLAG_TIME_KERNEL 2u /* record CUDA events around the projector kernel
                                   (not the layout transposes); read them back with
                                   ctp_plan_kernel_time_ms after the stream completes */

/* Flattened geometry: the f64 scalars of kernel_geom() plus the pose table. */
typedef struct ctp_geom {
  int32_t kind;       /* enum ctp_kind */
  int32_t num_views;  /* nv */
  int32_t num_rows;   /* nr */
  int32_t num_cols;   /* nc */
  int32_t num_x;      /* nx */
  int32_t num_y;      /* ny */
  int32_t num_z;      /* nz */
  int32_t reserved0;  /* must be 0 */
  double pixel_width;  /* pw */
  double pixel_height; /* ph */
  double center_row;   /* cr */
  double center_col;   /* cc */
  double sdd;          /* 1.0 unless cone (as kernel_geom sets it) */
  double x0, y0, z0;   /* lower grid corner = offset - n*h/2 (VolumeSpec.bounds) */
  double voxel_width;  /* hx (also the y pitch) */
  double voxel_height; /* hz */
  /* host pointer, num_views*15 doubles: per view src[3], c0[3], u[3], vax[3], w[3]
   * exactly as pose_table() returns them */
  const double* poses;
} ctp_geom;

typedef struct ctp_plan ctp_plan;

/* Library identity. */
int ctp_abi_version(void);
const char* ctp_status_string(int status);
/* Copies the last error message of the calling thread into buf (NUL-terminated). */
int ctp_last_error(char* buf, size_t buf_bytes);

/* Plan: validated geometry + per-view coefficient table resident on device
 * `device` (the current device when < 0).  Creation synchronises once. */
int ctp_plan_create(const ctp_geom* geom, int device, ctp_plan** plan_out);
int ctp_plan_destroy(ctp_plan* plan);
/* Shape queries (handy for bindings). */
int ctp_plan_shape(const ctp_plan* plan, int64_t* vol_elems, int64_t* sino_elems);

/* Device workspace needed by ctp_sf_forward (direction 0) or ctp_sf_back
 * (direction 1) for `batch` elements.  Pass at least this many bytes. */
size_t ctp_sf_workspace_bytes(const ctp_plan* plan, int direction, int batch);

/* y = A_SF x   (sf_forward_kernel, _kernels.py:650-663) */
int ctp_sf_forward(const ctp_plan* plan, const float* vol, float* sino, int batch,
                   void* workspace, size_t workspace_bytes, uint32_t flags,
                   void* stream);

/* x = A_SF^T y (sf_back_kernel, _kernels.py:666-763) */
int ctp_sf_back(const ctp_plan* plan, const float* sino, float* vol, int batch,
                void* workspace, size_t workspace_bytes, uint32_t flags,
                void* stream);

/* Duration (ms) of the projector kernel of the last CTP_FLAG_TIME_KERNEL call
 * in `direction` (0 forward, 1 back) on this plan.  Synchronises on the
 * recorded end event.  Returns CTP_ERR_INVALID_ARGUMENT if none was recorded. */
/* FBP back projection: the Ram-Lak ramp filter of
 * every detector row (pkg/src/ctproj/recon.py:39-61, linear convolution, the
 * reference's zero-padded FFT) times `scale`, fused with the layout change of
 * the back projection's input, then the SF back projection into vol.  With
 * scale = pi d^2 / (nv hx^2) this is fbp_parallel (recon.py:64-83).
 * Workspace: ctp_sf_workspace_bytes(plan, 1, batch). */
int ctp_sf_fbp_back(const ctp_plan* plan, const float* sino, float* vol, int batch, double scale,
                    void* workspace, size_t workspace_bytes, uint32_t flags, void* stream);
int ctp_plan_kernel_time_ms(const ctp_plan* plan, int direction, float* ms);

/* Siddon pair (exact ray-voxel line lengths, float64 like the reference):
 *   ctp_siddon_forward <- siddon_forward_kernel(vol, out, kind, src, c0, u, vax,
 *                         w, pw, ph, cr, cc, sdd, back, x0, y0, z0, hx, hz)
 *                         (pkg/src/ctproj/_kernels.py:191-208), called by
 *                         siddon_forward (pkg/src/ctproj/siddon.py:18-23);
 *   ctp_siddon_back    <- siddon_back_kernel(y, out, ...same...)
 *                         (_kernels.py:282-387), called by siddon_backproject
 *                         (siddon.py:26-31).
 * `back` is kernel_geom's parallel-beam ray back-off (circumscribed radius of
 * the grid plus one voxel width, _common.py:21-24); it only matters for
 * parallel geometry.  No workspace; same layouts, flags and contract as the
 * SF entry points.  Every geometry kind, modular included, is supported. */
int ctp_siddon_forward(const ctp_plan* plan, double back, const float* vol, float* sino,
                       int batch, uint32_t flags, void* stream);
int ctp_siddon_back(const ctp_plan* plan, double back, const float* sino, float* vol,
                    int batch, uint32_t flags, void* stream);

/* One-shot variants with the reference kernel's shape: they build a
 * temporary plan, allocate workspace stream-ordered, launch, and release.
 * They synchronise the stream once (plan upload) and are meant for FFI
 * callers that do not keep state. */
int ctp_sf_forward_oneshot(const ctp_geom* geom, const float* vol, float* sino,
                           int batch, void* stream);
int ctp_sf_back_oneshot(const ctp_geom* geom, const float* sino, float* vol,
                        int batch, void* stream);

/* ---- multi-GPU (north_star item 4; the reference has no multi-device path) ----
 *
 * One process per GPU.  Views are sharded over ranks: rank r holds a plan over
 * its contiguous view range [a_r, b_r) and the FULL grid.  The forward needs no
 * communication (ctp_sf_forward on the shard writes the rank's views).  The
 * back projection of the shard is fused with the reduction across ranks:
 *
 *   ctp_sf_back_sharded: x_r = sum over ranks of A_shard^T y_shard, restricted
 *   to rank r's z-slab [r*S, (r+1)*S), S = ceil(nz / nranks) (slices past nz
 *   are zero).  The partial volume is produced in z-chunks of
 *   CTP_BACK_ZCHUNK slices on `stream`; as soon as a chunk is done, its parts
 *   are ncclReduce'd (sum, fp32) to the ranks owning them on the
 *   communicator's own stream, overlapped with the next chunk's back
 *   projection.  Equivalent to one reduce-scatter of the whole partial volume.
 *   `stream` waits for the last reduction: stream-ordered, no host sync.
 *
 * NCCL is loaded at run time (dlopen of libnccl.so.2, reusing the copy torch
 * already loaded); the library has no link-time NCCL dependency.
 */
#define CTP_BACK_ZCHUNK 256

typedef struct ctp_dist ctp_dist;

/* Fills id (128 bytes, an ncclUniqueId) on the root rank; share the bytes
 * with the other ranks out of band (e.g. torch.distributed). */
int ctp_dist_unique_id(unsigned char* id, size_t id_bytes);
/* Communicator of `nranks` processes, this one being `rank`, on `device`. */
int ctp_dist_create(const unsigned char* id, size_t id_bytes, int nranks, int rank, int device,
                    ctp_dist** out);
int ctp_dist_destroy(ctp_dist* dist);
/* Slab owned by `rank`: first slice and slice count S (slices >= nz are padding). */
int ctp_dist_slab(const ctp_plan* plan, const ctp_dist* dist, int rank, int* z_first, int* z_count);
size_t ctp_sf_back_sharded_workspace_bytes(const ctp_plan* plan, const ctp_dist* dist, int batch);
/* sino: this rank's views [batch][nv_r][nr][nc]; slab: [batch][S][ny][nx]. */
int ctp_sf_back_sharded(const ctp_plan* plan, ctp_dist* dist, const float* sino, float* slab, int batch,
                        void* workspace, size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* CTPROJ_B200_H */
