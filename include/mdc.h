/*
 * mdc.h -- C-ABI of the B200-native mdcontour hot path (libmdc.so).
 *
 * Plain C: device pointers, sizes, scalars, cudaStream_t (passed as void*).
 * No torch types cross this boundary; the Python package (ctypes) and any
 * other FFI bind these entry points directly.  Every call is stream-ordered
 * on the stream passed in and returns 0 on success or a negative MDC_E*
 * code; mdc_last_error() describes the last failure on the calling thread.
 *
 * Memory ownership: the library never allocates or frees caller memory.
 * Scratch comes from caller-supplied workspaces sized by *_workspace_bytes().
 *
 * Reference seams replaced (upstream package `mdcontour`, file:line under
 * /root/reference/pkg/src/mdcontour):
 *   mdc_mls_field       <- _kernels.mean_field / affine_field / rigid_field
 *                          (_kernels.py:52-175) as dispatched by
 *                          field.compute_field (field.py:616-626), plus the
 *                          band epilogue render._band_indices (render.py:135-139)
 *   mdc_mls_snap        <- field._snap_control_pixels (field.py:388-412)
 *   mdc_layout_*        <- layout.layout_step / layout_run (layout.py:266-302),
 *                          bhtree.KdTree + repulsive_forces (bhtree.py:10-95),
 *                          _kernels.bh_forces (_kernels.py:178-230),
 *                          layout._spring_forces / _node_edge_forces /
 *                          clamp_factors (layout.py:160-256)
 *   mdc_pca             <- projection.pca_project numerics (projection.py:50-79)
 */
#ifndef MDC_H
#define MDC_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define MDC_API __attribute__((visibility("default")))
#else
#define MDC_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define MDC_OK 0
#define MDC_EINVAL (-22)
#define MDC_ENOMEM (-12)
#define MDC_ECUDA (-5)

/* MLS variants (field.py:29 VARIANTS minus "linear") */
#define MDC_MEAN 1
#define MDC_AFFINE 2
#define MDC_RIGID 3

/* arithmetic type of the MLS accumulation */
#define MDC_F32 0
#define MDC_F64 1

MDC_API const char *mdc_last_error(void);
MDC_API int mdc_version(void);

/* ------------------------------------------------------------------------ */
/* MLS field.
 *
 * Evaluates pixel rows [row0, row1) of a width x height raster whose pixel
 * centres are (field.py:127-131)
 *     x = x0 + (col + 0.5) * sx,   y = y1 - (row + 0.5) * sy
 * against n controls.  Inputs are centred exactly as compute_field does
 * (field.py:607-613): pc = positions - pm (fp64, n x 2 interleaved), and the
 * pixel coordinates are shifted by pm inside the kernel.
 *
 *   q      : n x d targets in the compute dtype, row stride ldq elements,
 *            centred by qm (affine/rigid), or the mean variant's displacement
 *            dq = qc - pc[:, axis[k]] (_kernels.py:52-67 `dqx, dqy`).
 *   qm     : d fp64 target means added back (field.py:646).
 *   axis   : mean variant only -- per channel, 0 adds vx, 1 adds vy.
 *   out    : element (k, r, c) at out[k*out_cs + (r-row0)*out_rs + c*out_ps].
 *   bands  : optional int32 floor(out/spacing[k]) (render.py:135-139),
 *            element (k, r, c) at bands[k*band_cs + (r-row0)*band_rs + c].
 *   nonfinite : optional device int32 counter += pixels with a non-finite
 *            channel (before snapping; mdc_mls_snap subtracts the pixels it
 *            overwrites), backing field.py:650-651's FieldError.
 * Rigid requires d == 2 (field.py:593-595 rejects single-channel rigid).
 */
typedef struct MdcMlsArgs {
    int32_t variant, dtype;
    int32_t width, height, row0, row1;
    int64_t n;
    int32_t d, ldq;
    double x0, y1, sx, sy;
    double pmx, pmy;
    double alpha, reg_eps;
    const double *pc;
    const void *q;
    const double *qm;
    const int32_t *axis;
    void *out;
    int64_t out_cs, out_rs, out_ps;
    int32_t *bands;
    int64_t band_cs, band_rs;
    const double *spacing;
    int32_t *nonfinite;
    /* tensor-core path (fp32 affine, d >= 8): scratch for the pre-arranged
     * hi/lo target image, mdc_mls_workspace_bytes(a) bytes; NULL or too small
     * selects the SIMT kernel.  flags: MDC_FLAG_NO_TC forces SIMT. */
    int32_t flags;
    void *workspace;
    size_t workspace_bytes;
    /* Fused band shading (render.py:142-148 render_discrete of channel k's
     * single-dimension field): optional uint32 RGBA8 (little-endian R,G,B,A
     * bytes) per pixel-channel with the bands' strides,
     * rgba = palette[floor(f / spacing[k]) mod palette_n]; needs spacing. */
    uint32_t *rgba;
    const uint32_t *palette;
    int32_t palette_n;
    /* optional: the frame centre pm (2 fp64, device, e.g. mdc_mls_prepare's
     * output); when set the kernels read it there instead of pmx / pmy, so
     * the caller need not copy it back to the host (no stream sync). */
    const double *pm;
} MdcMlsArgs;

#define MDC_FLAG_NO_TC 1
#define MDC_FLAG_TC_ONEPASS 2 /* A/B only: the experimental one-pass tensor-core kernel (mls_tc2.cu) */

MDC_API int mdc_mls_field(const MdcMlsArgs *a, void *stream);
MDC_API size_t mdc_mls_workspace_bytes(const MdcMlsArgs *a);

/* Input staging (field.py:607-613): from raw positions (n x 2) and targets
 * (n x d, fp64, device), compute pm (2) and qm (d) -- deterministic chunked
 * column means, identical on every device -- the centred controls pc
 * (n x 2 fp64) and the padded target block q (n x ldq, MDC_F32/MDC_F64):
 * qc = tvals - qm, or for MDC_MEAN dq = qc - pc[:, axis[k]] (_kernels.py:
 * 52-67); columns d..ldq-1 are zero.  workspace: mdc_mls_prepare_workspace_bytes. */
MDC_API size_t mdc_mls_prepare_workspace_bytes(int32_t d);
MDC_API int mdc_mls_prepare(int64_t n, int32_t d, const double *positions, const double *tvals, int32_t variant,
                            int32_t dtype, const int32_t *axis, int32_t ldq, double *pc, void *q, double *pm,
                            double *qm, void *workspace, size_t workspace_bytes, void *stream);

/* Snap (field.py:388-412): pixels of rows [row0,row1) whose centre lies at
 * squared distance < eps from control i (un-centred positions, fp64 decisions
 * with the reference's exact rounding sequence) take tvals[i] (n x d fp64,
 * raw targets); nearest control wins, lower index on exact ties.  Writes the
 * same out/bands layout as mdc_mls_field (dtype from a->dtype).  `pos` is the
 * un-centred n x 2 fp64 positions.  workspace must be
 * mdc_snap_workspace_bytes(width, rows) bytes and all-0xFF on first use; the
 * call leaves it all-0xFF again. */
MDC_API size_t mdc_snap_workspace_bytes(int32_t width, int32_t rows);
MDC_API int mdc_mls_snap(const MdcMlsArgs *a, const double *pos, const double *tvals, double eps,
                 void *workspace, void *stream);

/* ------------------------------------------------------------------------ */
/* Linear variant (field._linear_field, field.py:497-515): rows [row0,row1) of
 * the raster get the barycentric blend of the lowest-index covering triangle
 * (_kernels.rasterize_linear, _kernels.py:233-269), else the plane of the
 * nearest hull triangle (_kernels.extend_hull, _kernels.py:272-313).
 * pos (n x 2 fp64, un-centred), tvals (n x nch fp64), tris (ntri x 3 int32),
 * hull (nhull x 3 int32: u, v, triangle in field._hull_edges order).  out in
 * `dtype` with the MdcMlsArgs stride convention.  workspace:
 * mdc_linear_workspace_bytes(width, rows) bytes of int32 INT32_MAX on first
 * use; the call leaves it in that state. */
typedef struct MdcLinearArgs {
    int32_t width, height, row0, row1;
    double x0, y1, sx, sy;
    int64_t n, ntri;
    int32_t nch, dtype;
    const double *pos, *tvals;
    const int32_t *tris, *hull;
    int32_t nhull;
    void *out;
    int64_t out_cs, out_rs, out_ps;
    void *workspace;
} MdcLinearArgs;
MDC_API size_t mdc_linear_workspace_bytes(int32_t width, int32_t rows);
MDC_API int mdc_linear_field(const MdcLinearArgs *a, void *stream);

/* ------------------------------------------------------------------------ */
/* Isocontour rendering (render.py:91-148): per image, band shading and/or
 * anti-aliased contour lines with np.gradient gradients, fp64 compositing,
 * RGBA8 out (images x H x W x 4).  An image is `channels` planes (1: the
 * CLI's per-dimension render; 2: a two-channel field, bands summed and
 * coverage maxed over channels).  Plane (img, c) element (r, x) lives at
 * values[img*img_stride + c*cs + r*rs + x*ps].  colormap: ncolors x 4 fp64
 * already divided by 255 (render.py:78-82).  Optional coverage (float, images
 * x H x W) receives line_coverage.  Full frames (np.gradient needs the
 * neighbouring rows). */
#define MDC_RENDER_CONTOUR 0
#define MDC_RENDER_DISCRETE 1
#define MDC_RENDER_DISCRETE_CONTOUR 2
#define MDC_RENDER_ADAPTIVE 3  /* render.py:151-178, octaves -3..3 */
#define MDC_RENDER_GRADIENT 4  /* render.py:181-201, needs channels == 2 */
#define MDC_RENDER_TEXTURE 5   /* render.py:204-234, RGBA8 texture tex_h x tex_w */
typedef struct MdcRenderArgs {
    int32_t mode, dtype, width, height, nimg, channels;
    const void *values;
    int64_t img_stride, cs, rs, ps;
    const double *spacing;
    double line_width_px;
    int32_t line_color[4], background[4];
    const double *colormap;
    int32_t ncolors;
    uint8_t *out;
    float *coverage;
    int32_t gradient_corners[16];   /* c00, c10, c01, c11 RGBA */
    double adaptive_target_px;
    const uint8_t *texture;
    int32_t tex_w, tex_h;
} MdcRenderArgs;
MDC_API int mdc_render(const MdcRenderArgs *a, void *stream);

/* Point overlay (render.py:237-257): anti-aliased discs of radius r at the
 * n projected points (pix: device n x 2 fp64 pixel coordinates =
 * ViewportTransform.to_pixels), composited onto img (device H x W x 4 RGBA8,
 * in place) in point order.  color: HOST pointer to 4 ints (RGBA).
 * workspace: mdc_overlay_workspace_bytes(n, r) device bytes. */
MDC_API size_t mdc_overlay_workspace_bytes(int64_t n, double radius);
MDC_API int mdc_overlay_points(uint8_t *img, int32_t width, int32_t height, int64_t n, const double *pix,
                               double radius, const int32_t *color, void *workspace, size_t workspace_bytes,
                               void *stream);

/* ------------------------------------------------------------------------ */
/* One-to-one seam replacements of the reference's numba kernels (same
 * arguments and out-parameter convention as _kernels.py, DEVICE pointers,
 * fp64, the reference's own operation order).  npix pixels at (vx, vy),
 * n controls, out is npix x 2.
 *   mdc_mean_field   <- _kernels.mean_field   (_kernels.py:52-67)
 *   mdc_affine_field <- _kernels.affine_field (_kernels.py:70-124)
 *   mdc_rigid_field  <- _kernels.rigid_field  (_kernels.py:127-175)
 *   mdc_bh_forces    <- _kernels.bh_forces    (_kernels.py:178-230), int64
 *                       flat kd-tree arrays exactly as bhtree.KdTree holds them */
MDC_API int mdc_mean_field(int64_t npix, const double *vx, const double *vy, int64_t n, const double *px,
                           const double *py, const double *dqx, const double *dqy, double alpha,
                           double *out, void *stream);
MDC_API int mdc_affine_field(int64_t npix, const double *vx, const double *vy, int64_t n, const double *px,
                             const double *py, const double *qx, const double *qy, double alpha,
                             double reg_eps, double *out, void *stream);
MDC_API int mdc_rigid_field(int64_t npix, const double *vx, const double *vy, int64_t n, const double *px,
                            const double *py, const double *qx, const double *qy, double alpha, double *out,
                            void *stream);
/* mdc_rigid_field plus |f| (the rotation estimate's norm) per pixel in
 * norm_out (npix, device): the scalar rigid_mls (field.py:243-267) raises
 * DegenerateRotation where it is < 1e-12 instead of taking the per-pixel
 * mean fallback of _kernels.rigid_field. */
MDC_API int mdc_rigid_field_norm(int64_t npix, const double *vx, const double *vy, int64_t n,
                                 const double *px, const double *py, const double *qx, const double *qy,
                                 double alpha, double *out, double *norm_out, void *stream);
MDC_API int mdc_bh_forces(int64_t n, const double *points, const int64_t *perm, const int64_t *lo,
                          const int64_t *hi, const int64_t *left, const int64_t *right, const double *com,
                          const double *mass, const double *size, const double *bmin, const double *bmax,
                          double c, double eta, double theta, double *out, void *stream);

/* ------------------------------------------------------------------------ */
/* Constrained layout (layout.py:266-302).
 *
 * Topology (int32, device): csr_off (n+1), csr_tgt (2E) in the mesh's CSR
 * order; tris (T x 4, the 4th int unused padding) canonical CCW triples;
 * inc_off (n+1) + inc (3T) per-vertex incident (triangle << 2 | corner)
 * entries sorted by (corner, triangle) -- the accumulation order of the
 * reference's per-corner np.bincount passes (layout.py:240-255).
 * pos (n x 2 fp64) holds the input snapshot and receives the result.
 * temps (k fp64, device) is the per-step temperature sequence
 * t_i = t_{i-1} * lambda computed by the caller exactly as layout.py:284.
 */
typedef struct MdcLayoutArgs {
    int64_t n, ntri;
    int32_t leaf;
    double c, spring, dlen, eta, theta;
    const int32_t *csr_off, *csr_tgt, *tris, *inc_off, *inc;
    double *pos;
    void *workspace;
    size_t workspace_bytes;
    /* optional debug outputs of the LAST step (teacher-forced parity): */
    double *dbg_bh;     /* n x 2 Barnes-Hut force            */
    double *dbg_force;  /* n x 2 BH + spring + node-edge      */
    double *dbg_scale;  /* n clamp factor s                   */
    /* vertex partition for multi-GPU steps: this rank
     * updates the vertices at kd-tree leaf-order positions
     * [n*rank/world, n*(rank+1)/world) and writes 0.0 for every other vertex,
     * so a SUM all-reduce of pos across ranks reassembles the step exactly.
     * world <= 1: the whole mesh. */
    int32_t part_rank, part_world;
} MdcLayoutArgs;

typedef struct MdcLayoutPlan MdcLayoutPlan;

MDC_API size_t mdc_layout_workspace_bytes(int64_t n, int32_t leaf);
/* Creates a plan (host object) and uploads the kd-tree shape, which depends
 * only on (n, leaf) (bhtree.py:51-66), into the workspace.  The plan caches
 * CUDA graphs of the step. */
MDC_API int mdc_layout_plan_create(const MdcLayoutArgs *a, MdcLayoutPlan **plan, void *stream);
MDC_API int mdc_layout_plan_destroy(MdcLayoutPlan *plan);
/* k Jacobi steps; temps points at k device doubles.  use_graph=1 replays a
 * captured CUDA graph per step. */
MDC_API int mdc_layout_steps(MdcLayoutPlan *plan, int32_t k, const double *temps, int32_t use_graph,
                     void *stream);
/* Profiling: ONE eager step of the plan (same result as mdc_layout_steps
 * k=1) with CUDA events between its phases.  ms_out[5] = {axis sorts, tree
 * levels + centroids, BH traversal, BH task combine, local forces + clamp +
 * update}.  counts_out[4] (nullable) = {leaf-pair interactions incl. the
 * zero self terms, monopole interactions, node opening tests, warp lane
 * slots spent (32 per visited node + 32 per leaf-loop iteration)} over this
 * rank's points, from a separate instrumented traversal before the timed
 * step.  Synchronizes the stream. */
MDC_API int mdc_layout_profile(MdcLayoutPlan *plan, const double *temps, float *ms_out, int64_t *counts_out,
                               void *stream);
/* Peer-memory exchange for the vertex partition:
 * instead of zero-filling the non-owned vertices for a SUM all-reduce, every
 * rank's step kernel stores its owned vertices' new positions straight into
 * ALL ranks' next-parity position buffers (NVLink stores into buffers mapped
 * with mdc_ipc_open).  peers0[r] / peers1[r] = rank r's parity-0 / parity-1
 * position buffer (n x 2 fp64) as mapped in this process; peers0[rank] must
 * be the plan's `pos`, peers1[rank] becomes its second buffer; 2 <= world
 * <= 8 = part_world.  Steps then run with mdc_layout_step_parity, and the
 * caller orders them across ranks (stream sync + host barrier per step). */
MDC_API int mdc_layout_set_peers(MdcLayoutPlan *plan, int32_t world, double *const *peers0, double *const *peers1);
/* One step reading the parity-p buffer (0 = pos, 1 = the second buffer) and
 * writing the other one; no copy-back.  mdc_layout_reset_counter restarts
 * the temps index (the step count into `temps`). */
MDC_API int mdc_layout_step_parity(MdcLayoutPlan *plan, int32_t parity, const double *temps, int32_t use_graph,
                                   void *stream);
/* Vertex-partitioned plans (part_world > 1), all-gather exchange (SURVEY.md
 * §8e "positions NCCL-allgathered once per iteration"): after
 * mdc_layout_set_gather(plan, send) -- before the first step -- each step
 * writes this rank's owned slice (leaf order n*r/w .. n*(r+1)/w of the step's
 * kd-tree) packed into send (ceil(n/w) x 2 fp64, device) instead of pos; the
 * caller all-gathers the send buffers of all ranks into recv (w x chunk x 2,
 * rank-major, e.g. ncclAllGather) and mdc_layout_scatter(plan, recv, chunk)
 * writes every vertex's new position into pos through the step's
 * permutation.  Bit-identical to the single-GPU step. */
MDC_API int mdc_layout_set_gather(MdcLayoutPlan *p, double *send);
MDC_API int mdc_layout_scatter(MdcLayoutPlan *p, const double *recv, int64_t chunk, void *stream);
MDC_API int mdc_layout_reset_counter(MdcLayoutPlan *plan, void *stream);
/* Inter-process device buffers (cudaIpc): allocate + 64-byte handle, open a
 * peer's handle in this process, close an opened mapping, free an allocation. */
MDC_API int mdc_ipc_alloc(size_t bytes, void **ptr, void *handle64);
MDC_API int mdc_ipc_open(const void *handle64, void **ptr);
MDC_API int mdc_ipc_close(void *ptr);
MDC_API int mdc_ipc_free(void *ptr);
/* clamp_factors (layout.py:160-184) for an arbitrary displacement field:
 * s_out[i] = largest factor in [0, 1] keeping node i eta clear of the three
 * mid-segment limiting lines of each incident triangle (inc_off/inc as in
 * MdcLayoutArgs) when it moves by disp[i].  Same operations as the step. */
MDC_API int mdc_layout_clamp_factors(int64_t n, const double *pos, const double *disp, const int32_t *tris,
                                     const int32_t *inc_off, const int32_t *inc, double eta, double *s_out,
                                     void *stream);
/* Barnes-Hut repulsion alone for positions pts (bhtree.py:69-95). */
MDC_API int mdc_layout_repulsion(MdcLayoutPlan *plan, const double *pts, double *out, void *stream);
/* kd-tree of pts: node arrays (count = mdc_layout_node_count) copied out. */
MDC_API int64_t mdc_layout_node_count(const MdcLayoutPlan *plan);
MDC_API int mdc_layout_kdtree(MdcLayoutPlan *plan, const double *pts, int32_t *perm, int32_t *lo,
                      int32_t *hi, int32_t *left, int32_t *right, double *com, double *mass,
                      double *size, double *bmin, double *bmax, void *stream);

/* ------------------------------------------------------------------------ */
/* PCA (projection.py:50-79): x is n x d fp64 row-major on device.  Outputs:
 * mean (d), cov (d x d), eigenvalues (2, descending, clipped at 0), axes
 * (2 x d, sign rule of projection.py:71-74), positions (n x 2). */
MDC_API size_t mdc_pca_workspace_bytes(int64_t n, int32_t d);
MDC_API int mdc_pca(int64_t n, int32_t d, const double *x, double *mean, double *cov, double *eigenvalues,
            double *axes, double *positions, void *workspace, void *stream);

/* ------------------------------------------------------------------------ */
/* Roofline helpers: time-free peak kernels (the caller times them). */
MDC_API int mdc_peak_ffma(float *sink, int32_t blocks, int32_t iters, void *stream);
MDC_API int mdc_peak_dfma(double *sink, int32_t blocks, int32_t iters, void *stream);
MDC_API int mdc_num_sms(void);
/* Stream-ordered strided copy (cudaMemcpy2DAsync, any direction): `height`
 * rows of `width_bytes`; used to deliver a row band of every channel plane
 * to pinned host memory in one call while the next band computes. */
MDC_API int mdc_copy_2d_async(void *dst, size_t dpitch, const void *src, size_t spitch, size_t width_bytes,
                              size_t height, void *stream);

#ifdef __cplusplus
}
#endif
#endif
