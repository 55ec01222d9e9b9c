/*
 * difform_gpu.h — C-ABI boundary of the B200-native dense diffeomorphic
 * matching path (FireANTs direct-mode loop, reference "difform").
 *
 * Every entry point here replaces one function of the reference C++ API in
 * /root/reference/proj/include/difform/ (cited per function).  The reference
 * has no FFI of its own: its boundary is the header API, so the C-ABI keeps
 * the same argument meaning with plain pointers and sizes:
 *
 *   - grids are described by dfm_grid (== difform::GridMeta, core.hpp:13-23);
 *   - images are x-fastest arrays of voxel_count doubles (ScalarImage::data,
 *     core.hpp:36-42); label maps int32 (LabelImage, core.hpp:44-50);
 *   - vector fields are interleaved AoS doubles, ndim per voxel, voxel units
 *     of their own grid (VectorField::data, core.hpp:54-64);
 *   - every buffer argument is a HOST pointer; the library stages it through
 *     pinned memory into device SoA planes of the context precision and
 *     copies results back (no torch types, no device pointers in the
 *     host-level calls).  The dfm_dev_* calls at the end take DEVICE pointers
 *     for callers whose data already lives in HBM.
 *
 * Errors mirror the reference exception classes:
 *   DFM_E_INVALID   <-> std::invalid_argument (validation, grid mismatch)
 *   DFM_E_NUMERICAL <-> std::runtime_error    (non-finite loss/step, fold)
 *   DFM_E_CUDA      <-> device failure (no reference counterpart)
 * The message of the last failure on the calling host thread is returned by
 * dfm_last_error().
 *
 * Threading: a dfm_ctx owns one CUDA stream, a workspace arena and a CUDA
 * graph cache; it must be used by one host thread at a time.  Use one
 * context per thread for the reference's concurrent sweep
 * (pipeline.cpp:287-301).  Results never depend on the thread count.
 */
#ifndef DIFFORM_GPU_H
#define DIFFORM_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DFM_ABI_VERSION 1

#if defined(__GNUC__)
#define DFM_API __attribute__((visibility("default")))
#else
#define DFM_API
#endif

typedef enum {
    DFM_OK = 0,
    DFM_E_INVALID = 1,
    DFM_E_NUMERICAL = 2,
    DFM_E_CUDA = 3
} dfm_status;

/* arithmetic/storage type of the device path */
typedef enum { DFM_PREC_F32 = 0, DFM_PREC_F64 = 1 } dfm_precision;
/* element type of host image/field buffers handed to dfm_register */
typedef enum { DFM_HOST_F32 = 0, DFM_HOST_F64 = 1 } dfm_host_dtype;
/* difform::LossKind (affine.hpp:9) */
typedef enum { DFM_LOSS_SSD = 0, DFM_LOSS_LNCC = 1, DFM_LOSS_DICE = 2 } dfm_loss;
/* difform::RegMode (pipeline.hpp:23) */
typedef enum { DFM_MODE_DIRECT = 0, DFM_MODE_SVF = 1 } dfm_mode;
/* difform::RegInit alternatives (pipeline.hpp:62) */
typedef enum { DFM_INIT_NONE = 0, DFM_INIT_AFFINE = 1, DFM_INIT_FIELD = 2 } dfm_init_kind;

/* difform::GridMeta (core.hpp:13-23).  ndim 2 uses dims[2] == 1. */
typedef struct {
    int32_t ndim;
    int64_t dims[3];
    double spacing[3];
    double origin[3];
} dfm_grid;

/* difform::RegistrationConfig (pipeline.hpp:25-41) */
typedef struct {
    int32_t loss;        /* dfm_loss */
    int32_t lncc_radius;
    double eta;
    double sigma_grad;
    double sigma_warp;
    int32_t use_jac;
    int32_t mode;        /* dfm_mode: direct (the hot path) or svf (exp_map + pullback) */
    int32_t svf_M;
    double beta1;
    double beta2;
    double eps_adam;
    double step_cap;
    int32_t conv_window;
    double conv_tol;
    uint64_t seed;
} dfm_config;

/* difform::IterationRecord (pipeline.hpp:45-53) */
typedef struct {
    int32_t scale_index;
    double scale;
    int32_t iter;
    int64_t global_iter;
    double loss;
    double max_step;
    double wall_ms;
} dfm_iter_record;

/* difform::RegInit (pipeline.hpp:62): none, AffineTransform (affine.hpp:12-16)
 * or a displacement field on the full or the coarsest working grid. */
typedef struct {
    int32_t kind;        /* dfm_init_kind */
    int32_t affine_ndim;
    double A[9];         /* row-major, ndim x ndim used */
    double t[3];
    dfm_grid field_grid; /* DFM_INIT_FIELD: grid of `field` */
    const double* field; /* DFM_INIT_FIELD: AoS doubles (host) */
} dfm_init;

/* difform::AffineResult (affine.hpp:18-23): best-loss iterate of
 * affine_register (the last finite one on divergence). */
typedef struct {
    int32_t ndim;
    double A[9];         /* row-major, ndim x ndim used */
    double t[3];
    double loss;
    int32_t diverged;
    int64_t iterations;
} dfm_affine_result;

/* difform::RegionOverlap (analysis.hpp:46-59) */
typedef struct {
    int32_t label;
    int32_t has_to, has_fn, has_fp;
    int64_t fixed_count;   /* |T_r| */
    int64_t warped_count;  /* |S_r| */
    int64_t intersection;  /* |S_r n T_r| */
    double to, mo, fn, fp, vs;
} dfm_region_overlap;

/* difform::OverlapReport aggregates (analysis.hpp:61-65) */
typedef struct {
    double to_mean, mo_mean, fn_mean, fp_mean, vs_mean;
    double to_klein, mo_klein, fn_klein, fp_klein, vs_klein;
    int64_t n_regions;     /* regions in the report (may exceed the capacity passed) */
} dfm_overlap_summary;

/* Result summary of dfm_register: difform::RunLog (pipeline.hpp:55-60). */
typedef struct {
    int64_t n_records;   /* records written (<= capacity passed in)   */
    int64_t n_total;     /* records produced (may exceed capacity)     */
    double final_loss;
    double final_singularity_fraction;
    double total_ms;
} dfm_runlog;

typedef struct dfm_ctx dfm_ctx;

/* ---- library / context ------------------------------------------------- */
DFM_API int dfm_abi_version(void);
/* RegistrationConfig{} defaults (pipeline.hpp:25-41). */
DFM_API void dfm_config_defaults(dfm_config* cfg);
/* Creates a context on `device` computing in `precision` (dfm_precision). */
DFM_API dfm_status dfm_ctx_create(int device, int precision, dfm_ctx** out);
DFM_API void dfm_ctx_destroy(dfm_ctx* ctx);
DFM_API int dfm_ctx_precision(const dfm_ctx* ctx);
/* Copies the thread's last error message; returns its full length. */
DFM_API size_t dfm_last_error(char* buf, size_t cap);
/* The context's CUDA stream (a cudaStream_t), for callers that time or order
 * work around the library's launches with their own CUDA events. */
DFM_API void* dfm_ctx_stream(dfm_ctx* ctx);
/* Kernel launches issued by this context since creation (evidence count). */
DFM_API int64_t dfm_ctx_launch_count(const dfm_ctx* ctx);

/* ---- core.hpp ---------------------------------------------------------- */
/* validate_meta (core.cpp:26-37) */
DFM_API dfm_status dfm_validate_grid(const dfm_grid* g);
/* output grid of downsample_image (core.cpp:58-74) */
DFM_API dfm_status dfm_downsample_grid(const dfm_grid* g, const double factor[3], dfm_grid* out);
/* downsample_image (core.hpp:86-87, core.cpp:58-96) */
DFM_API dfm_status dfm_downsample_image(dfm_ctx* ctx, const dfm_grid* g, const double* img,
                                const double factor[3], dfm_grid* out_grid, double* out);

/* ---- interp.hpp -------------------------------------------------------- */
/* sample_linear + sample_linear_gradient (interp.hpp:11-17) at npts points
 * (xyz triples); grads may be NULL. */
DFM_API dfm_status dfm_sample_linear_points(dfm_ctx* ctx, const dfm_grid* g, const double* img,
                                    int64_t npts, const double* points, double* values,
                                    double* grads);
/* sample_field + sample_field_jacobian (interp.hpp:18-24, interp.cpp:188-227)
 * of an AoS field at npts points (xyz triples): values 3 per point (ndim
 * used), jac 9 per point row-major J[c][a] = d f_c / d x_a (may be NULL). */
DFM_API dfm_status dfm_sample_field_points(dfm_ctx* ctx, const dfm_grid* g, const double* field,
                                           int64_t npts, const double* points, double* values,
                                           double* jac);
/* warp_image (interp.hpp:28) */
DFM_API dfm_status dfm_warp_image(dfm_ctx* ctx, const dfm_grid* g, const double* img,
                          const double* phi, double* out);
/* warp_labels (interp.hpp:31) */
DFM_API dfm_status dfm_warp_labels(dfm_ctx* ctx, const dfm_grid* g, const int32_t* labels,
                           const double* phi, int32_t* out);
/* compose (interp.hpp:35): out = u_psi + lerp(u_phi)(x + u_psi) */
DFM_API dfm_status dfm_compose(dfm_ctx* ctx, const dfm_grid* g, const double* phi,
                       const double* psi, double* out);
/* ---- affine.hpp: pre-alignment (the step before the diffeomorphic path) ----- */
/* affine_to_field (affine.hpp:29-30): u(x) = (A - I) x + t on grid g. */
DFM_API dfm_status dfm_affine_to_field(dfm_ctx* ctx, const dfm_grid* g, const double A[9],
                                       const double t[3], double* out);
/* affine_param_gradient (affine.hpp:43-46, affine.cpp:95-122): loss of the
 * affine warp u = S^-1 (A S x + t) - x on a working-scale pair and its
 * parameter gradient dL/dA (row-major), dL/dt. */
DFM_API dfm_status dfm_affine_param_gradient(dfm_ctx* ctx, const dfm_grid* g,
                                             const double* fixed, const double* moving,
                                             int loss, const double A[9], const double t[3],
                                             const double scale_to_full[3], int lncc_radius,
                                             double* value, double dA[9], double dt[3]);
/* affine_register (affine.hpp:25-30, affine.cpp:124-183): multi-scale Adam
 * (beta 0.9/0.999, eps 1e-8) on (A, t) from identity; best-loss iterate;
 * non-finite loss -> diverged (no error); |det A| < 1e-3 -> DFM_E_NUMERICAL. */
DFM_API dfm_status dfm_affine_register(dfm_ctx* ctx, const dfm_grid* g, const double* fixed,
                                       const double* moving, int loss, const double* scales,
                                       const int32_t* iters, int32_t nscales, double eta,
                                       int lncc_radius, dfm_affine_result* out);

/* exp_map (diffeo.hpp:19-20, diffeo.cpp:66-77): v / 2^M, then M
 * self-compositions.  M < 0 -> DFM_E_INVALID. */
DFM_API dfm_status dfm_exp_map(dfm_ctx* ctx, const dfm_grid* g, const double* v, int M,
                               double* out);
/* svf_pullback (diffeo.hpp:22-26, diffeo.cpp:79-167): the discrete adjoint of
 * exp_map applied to the cotangent grad_phi.  The reference's serial scatter
 * is a stable-sorted gather on the device: same per-node summation order,
 * bit-stable across runs. */
DFM_API dfm_status dfm_svf_pullback(dfm_ctx* ctx, const dfm_grid* g, const double* v,
                                    const double* grad_phi, int M, double* out);
/* jacobian (interp.hpp:49, interp.cpp:291-328): per-voxel J = I + central
 * differences, ndim*ndim row-major doubles per voxel. */
DFM_API dfm_status dfm_jacobian(dfm_ctx* ctx, const dfm_grid* g, const double* phi, double* out);
/* jacobian_det (interp.hpp:50) */
DFM_API dfm_status dfm_jacobian_det(dfm_ctx* ctx, const dfm_grid* g, const double* phi, double* out);
/* gaussian_smooth / gaussian_smooth_field (interp.hpp:54-57) */
DFM_API dfm_status dfm_gaussian_smooth(dfm_ctx* ctx, const dfm_grid* g, const double* img,
                               const double sigma[3], double* out);
DFM_API dfm_status dfm_gaussian_smooth_field(dfm_ctx* ctx, const dfm_grid* g, const double* f,
                                     const double sigma[3], double* out);
/* upsample_field (linear), resample_field_linear, resample_displacement
 * (interp.hpp:65-75) */
DFM_API dfm_status dfm_upsample_field(dfm_ctx* ctx, const dfm_grid* g, const double* phi,
                              const dfm_grid* new_grid, double* out);
/* upsample_field with UpsampleMethod::cubic (interp.hpp:65-67,
 * interp.cpp:59-101): Catmull-Rom, the reference's folding demonstration. */
DFM_API dfm_status dfm_upsample_field_cubic(dfm_ctx* ctx, const dfm_grid* g, const double* phi,
                                            const dfm_grid* new_grid, double* out);
DFM_API dfm_status dfm_resample_field_linear(dfm_ctx* ctx, const dfm_grid* g, const double* f,
                                     const dfm_grid* new_grid, double* out);
DFM_API dfm_status dfm_resample_displacement(dfm_ctx* ctx, const dfm_grid* g, const double* phi,
                                     const dfm_grid* new_grid, double* out);

/* ---- similarity.hpp ---------------------------------------------------- */
/* ssd_eval / lncc_eval (similarity.hpp:17-24).  The moving image may live on
 * its own grid; phi must be on the fixed grid.  grad may be NULL. */
DFM_API dfm_status dfm_ssd_eval(dfm_ctx* ctx, const dfm_grid* fixed_grid, const double* fixed,
                        const dfm_grid* moving_grid, const double* moving,
                        const double* phi, double* value, double* grad);
DFM_API dfm_status dfm_lncc_eval(dfm_ctx* ctx, const dfm_grid* fixed_grid, const double* fixed,
                         const dfm_grid* moving_grid, const double* moving,
                         const double* phi, int window_radius, double* value, double* grad);
/* dice_soft_eval (similarity.hpp:27-28): masks must lie in [0,1]. */
DFM_API dfm_status dfm_dice_eval(dfm_ctx* ctx, const dfm_grid* fixed_grid, const double* fixed,
                         const dfm_grid* moving_grid, const double* moving,
                         const double* phi, double* value, double* grad);

/* ---- optim.hpp --------------------------------------------------------- */
/* adam_step (optim.hpp:23): m, nu updated in place, *t advanced. */
DFM_API dfm_status dfm_adam_step(dfm_ctx* ctx, const dfm_grid* g, double* m, double* nu,
                         int64_t* t, double beta1, double beta2, double eps,
                         const double* v, double* dir);
/* sgd_step (optim.hpp:27-29, optim.cpp:44-57): momentum 0 returns v and
 * leaves mu; otherwise mu <- momentum*mu + v (in place) and out = mu. */
DFM_API dfm_status dfm_sgd_step(dfm_ctx* ctx, const dfm_grid* g, double* mu, const double* v,
                                double momentum, double* out);
/* upsample_state (optim.hpp:31) */
DFM_API dfm_status dfm_upsample_state(dfm_ctx* ctx, const dfm_grid* g, const double* m,
                              const double* nu, const dfm_grid* new_grid, double* m_out,
                              double* nu_out);

/* ---- diffeo.hpp -------------------------------------------------------- */
/* eulerian_direction (diffeo.hpp:10-11) */
DFM_API dfm_status dfm_eulerian_direction(dfm_ctx* ctx, const dfm_grid* g, const double* grad,
                                  const double* phi, int use_jac, double* out);
/* apply_update (diffeo.hpp:16-17) */
DFM_API dfm_status dfm_apply_update(dfm_ctx* ctx, const dfm_grid* g, const double* phi,
                            const double* v, double eta, double sigma_warp, double cap,
                            double* out);

/* ---- analysis.hpp ------------------------------------------------------ */
/* singularity_fraction (analysis.hpp:40) */
DFM_API dfm_status dfm_singularity_fraction(dfm_ctx* ctx, const dfm_grid* g, const double* phi,
                                    double* fraction);

/* ---- pipeline.hpp ------------------------------------------------------ */
/* validate_config / validate_schedule (pipeline.hpp:21,43, pipeline.cpp:83-119):
 * DFM_E_INVALID with the reference's message. */
DFM_API dfm_status dfm_validate_config(const dfm_config* cfg);
DFM_API dfm_status dfm_validate_schedule(const double* scales, const int32_t* iterations,
                                         int32_t nscales);
/* register_images, direct mode (pipeline.hpp:70-73, pipeline.cpp:121-224).
 * fixed/moving: host arrays of `image_dtype` (dfm_host_dtype) on grid g.
 * out_field: host AoS array of `field_dtype` (voxel_count*ndim) or NULL.
 * records: capacity `max_records`; log->n_total says how many were made. */
DFM_API dfm_status dfm_register(dfm_ctx* ctx, const dfm_grid* g, const void* fixed,
                        const void* moving, int image_dtype, const dfm_config* cfg,
                        const double* scales, const int32_t* iterations, int32_t nscales,
                        const dfm_init* init, void* out_field, int field_dtype,
                        dfm_iter_record* records, int64_t max_records, dfm_runlog* log);

/* ---- device-resident entry points ------------------------------------- */
/* Same as dfm_register but fixed/moving are DEVICE arrays of the context
 * precision (float or double, voxel_count each) and the result field stays on
 * the device as three SoA planes of the context precision (out_soa_field:
 * 3*voxel_count elements, x-plane then y then z; may be NULL).  No host
 * staging is done except the per-scale loss log readback. */
DFM_API dfm_status dfm_dev_register(dfm_ctx* ctx, const dfm_grid* g, const void* d_fixed,
                            const void* d_moving, const dfm_config* cfg,
                            const double* scales, const int32_t* iterations,
                            int32_t nscales, void* d_out_soa_field,
                            dfm_iter_record* records, int64_t max_records, dfm_runlog* log);

/* ---- evaluation epilogue (analysis.hpp, interp.hpp) -------------------- */
/* overlap_report (analysis.hpp:67, analysis.cpp:169-247): per-region and
 * aggregate TO/MO/FN/FP/VS of a warped vs a fixed label map; regions in
 * ascending label order, at most max_regions written.  Labels above 2^24 ->
 * DFM_E_INVALID (MHD label maps are MET_SHORT).  Grid mismatch -> DFM_E_INVALID. */
DFM_API dfm_status dfm_overlap_report(dfm_ctx* ctx, const dfm_grid* warped_grid,
                                      const int32_t* warped, const dfm_grid* fixed_grid,
                                      const int32_t* fixed, dfm_overlap_summary* out,
                                      dfm_region_overlap* regions, int64_t max_regions);
/* Same on device label maps (no host round trip of the volumes). */
DFM_API dfm_status dfm_dev_overlap_report(dfm_ctx* ctx, const dfm_grid* g,
                                          const int32_t* d_warped, const int32_t* d_fixed,
                                          dfm_overlap_summary* out, dfm_region_overlap* regions,
                                          int64_t max_regions);
/* warp_labels (interp.hpp:33) on device buffers: d_field_soa is a 3-plane SoA
 * field in the context precision (as dfm_dev_register writes it). */
DFM_API dfm_status dfm_dev_warp_labels(dfm_ctx* ctx, const dfm_grid* g, const int32_t* d_labels,
                                       const void* d_field_soa, int32_t* d_out);
/* landmark_error (analysis.hpp:77-79, analysis.cpp:249-283): fixed-space
 * points (mm, n x 3) mapped through phi (AoS doubles on phi_grid == fixed
 * grid) into the moving frame; Euclidean mm distances to the moving points. */
DFM_API dfm_status dfm_landmark_error(dfm_ctx* ctx, const dfm_grid* fixed_grid,
                                      const dfm_grid* moving_grid, const dfm_grid* phi_grid,
                                      const double* phi, int64_t n, const double* fixed_mm,
                                      const double* moving_mm, double* distances, double* mean,
                                      double* max);

/* ---- hyperparameter sweep (pipeline.hpp:75-104, pipeline.cpp:226-313) -- */
/* difform::SweepPair: images on one grid (host AoS doubles); labels optional
 * (NULL) unless the metric is overlap. */
typedef struct {
    const dfm_grid* grid;
    const double* fixed;
    const double* moving;
    const int32_t* fixed_labels;
    const int32_t* moving_labels;
} dfm_sweep_pair;

/* difform::SweepRow */
typedef struct {
    double eta, sigma_warp, sigma_grad;
    double metric_mean, metric_sd;
    double wall_ms;
    int32_t failed;
    int32_t computed;     /* 1 for the rows of this call's shard */
    char error[256];
} dfm_sweep_row;

typedef enum { DFM_SWEEP_LOSS = 0, DFM_SWEEP_OVERLAP = 1 } dfm_sweep_metric;

/* sweep: grid eta x sigma_warp x sigma_grad (config k = (ei * n_sw + wi) *
 * n_sg + gi, as pipeline.cpp:254-257); each config registers every pair;
 * metric = final loss or overlap TO mean (analysis.cpp), mean and SD over the
 * pairs; failures are recorded per row.  Configs run concurrently on
 * `ndevices` GPUs x `workers_per_device` contexts (the reference's worker
 * threads, one CUDA stream each); pairs are uploaded once per context.  Only
 * configs k = shard_begin + j * shard_step are computed (multi-process
 * sharding; 0, 1 = all).  rows has n_eta * n_sw * n_sg entries. */
DFM_API dfm_status dfm_sweep(const int* devices, int ndevices, int workers_per_device,
                             int precision, const dfm_sweep_pair* pairs, int npairs,
                             const dfm_config* base, const double* scales,
                             const int32_t* iterations, int32_t nscales, const double* etas,
                             int n_eta, const double* sigma_warps, int n_sw,
                             const double* sigma_grads, int n_sg, int metric,
                             int64_t shard_begin, int64_t shard_step, dfm_sweep_row* rows);

/* ---- MetaImage I/O (io.hpp; io.cpp:117-328 format) ---------------------- */
typedef enum { DFM_MET_OTHER = -1, DFM_MET_FLOAT = 0, DFM_MET_SHORT = 1 } dfm_met_type;
typedef struct {
    dfm_grid grid;
    int32_t element_type;         /* dfm_met_type */
    int32_t channels;
    char element_type_name[32];
    char raw_path[1024];          /* ElementDataFile resolved against the header dir */
} dfm_mhd_info;
/* read_mhd_header (io.cpp:152-216); errors "path: byte N: ..." -> DFM_E_INVALID */
DFM_API dfm_status dfm_mhd_read_header(const char* path, dfm_mhd_info* out);
/* write_image_mhd / read_image_mhd (io.cpp:245-269): MET_FLOAT, 1 channel.
 * Readers: out == NULL queries the grid; capacity in elements. */
DFM_API dfm_status dfm_mhd_write_image(const char* path, const dfm_grid* g, const double* img);
DFM_API dfm_status dfm_mhd_read_image(const char* path, dfm_grid* g, double* out,
                                      int64_t capacity);
/* write_labels_mhd / read_labels_mhd (io.cpp:271-304): MET_SHORT */
DFM_API dfm_status dfm_mhd_write_labels(const char* path, const dfm_grid* g,
                                        const int32_t* labels);
DFM_API dfm_status dfm_mhd_read_labels(const char* path, dfm_grid* g, int32_t* out,
                                       int64_t capacity);
/* write_field_mhd / read_field_mhd (io.cpp:306-328): MET_FLOAT, ndim channels */
DFM_API dfm_status dfm_mhd_write_field(const char* path, const dfm_grid* g, const double* field);
DFM_API dfm_status dfm_mhd_read_field(const char* path, dfm_grid* g, double* out,
                                      int64_t capacity);
/* Streaming device feed: an MET_FLOAT image straight into HBM (context
 * precision) through pinned double-buffered chunks; d_out == NULL queries the
 * grid.  And a device SoA field (as dfm_dev_register writes it) to .mhd/.raw. */
DFM_API dfm_status dfm_dev_load_image_mhd(dfm_ctx* ctx, const char* path, dfm_grid* g,
                                          void* d_out);
DFM_API dfm_status dfm_dev_save_field_mhd(dfm_ctx* ctx, const char* path, const dfm_grid* g,
                                          const void* d_field_soa);

/* ---- z-slab decomposition (BASELINE config 4) ------------ */
/* Owned planes [zlo, zhi) and halo depths (hlo, hhi) of slab `part` of
 * `nparts` over nz planes with halo H: out = {zlo, zhi, hlo, hhi}. */
DFM_API dfm_status dfm_slab_bounds(int64_t nz, int part, int nparts, int halo, int64_t out[4]);
/* Halo depth (planes) the iteration needs for this config on grid g. */
DFM_API int dfm_slab_halo(const dfm_config* cfg, const dfm_grid* g);
/* 128-byte NCCL unique id for a slab group (rank 0 creates, all ranks use). */
DFM_API dfm_status dfm_slab_unique_id(unsigned char id[128]);
/* register_images (direct mode, LNCC) on a z-slab decomposition: the z
 * planes are split into `world` slabs; this process owns slab `rank` on the
 * context's device and exchanges halo planes with its neighbours over NCCL
 * (nccl_id from dfm_slab_unique_id) inside the captured iteration graphs; the
 * loss is all-reduced every iteration so the convergence monitor is global.
 * With world == 1, `emulate` > 1 splits the volume into that many slabs on
 * this one device and exchanges halos by device copies (same kernels, same
 * exchange plan).  d_fixed / d_moving: the FULL volumes (context precision)
 * on this device.  d_out_soa_field: 3 component planes of this process's
 * owned full-resolution planes (emulation: the whole volume); out_zlo/zhi
 * return them. */
DFM_API dfm_status dfm_dev_register_slab(dfm_ctx* ctx, const dfm_grid* g, const void* d_fixed,
                                         const void* d_moving, const dfm_config* cfg,
                                         const double* scales, const int32_t* iterations,
                                         int32_t nscales, int rank, int world,
                                         const unsigned char* nccl_id, int emulate,
                                         void* d_out_soa_field, int64_t* out_zlo,
                                         int64_t* out_zhi, dfm_iter_record* records,
                                         int64_t max_records, dfm_runlog* log);

/* A caller-provided transport for the slab exchange (no reference
 * counterpart): the slab loop's three collective steps — halo exchange with
 * the z neighbours, global sums/maxima for the loss and the convergence
 * monitor, and the gather of owned blocks at scale changes — go through these
 * host callbacks on host-staged (pinned) buffers.  It lets a slab
 * decomposition run across processes without NCCL (e.g. two processes on one
 * GPU, or a CPU-side messaging layer); the NCCL path keeps its device-side
 * collectives inside the captured iteration graphs.  Each callback returns 0
 * on success.  Every rank makes the same sequence of calls. */
typedef struct dfm_slab_transport {
    void* user;
    /* send `send_bytes` to rank `peer` and receive `recv_bytes` from it */
    int (*sendrecv)(void* user, int peer, const void* sendbuf, int64_t send_bytes,
                    void* recvbuf, int64_t recv_bytes);
    /* in-place element-wise sum over all ranks of n doubles */
    int (*allreduce_sum_f64)(void* user, double* buf, int64_t n);
    /* in-place element-wise maximum over all ranks of n unsigned 64-bit ints */
    int (*allreduce_max_u64)(void* user, uint64_t* buf, int64_t n);
    /* every rank's block (send_bytes; rank r contributes counts[r] bytes) into
     * recvbuf, concatenated in rank order */
    int (*allgather)(void* user, const void* sendbuf, int64_t send_bytes, void* recvbuf,
                     const int64_t* counts);
} dfm_slab_transport;

/* dfm_dev_register_slab over a caller transport: the same plan, kernels and
 * call sequence as the NCCL path (world > 1, this process = slab `rank`),
 * with every collective host-staged through `tp`. */
DFM_API dfm_status dfm_dev_register_slab_tp(dfm_ctx* ctx, const dfm_grid* g, const void* d_fixed,
                                            const void* d_moving, const dfm_config* cfg,
                                            const double* scales, const int32_t* iterations,
                                            int32_t nscales, int rank, int world,
                                            const dfm_slab_transport* tp, void* d_out_soa_field,
                                            int64_t* out_zlo, int64_t* out_zhi,
                                            dfm_iter_record* records, int64_t max_records,
                                            dfm_runlog* log);

/* Timing hook for benchmarks: per-kernel-class accumulated device time (ms)
 * and launch counts over the last dfm_register/dfm_dev_register call when
 * profiling is enabled with dfm_ctx_set_profiling(ctx, 1).  Class ids:
 * 0 lncc/ssd forward, 1 lncc backward, 2 smooth+adam, 3 compose+smooth,
 * 4 monitor, 5 pyramid (down/upsample), 6 epilogue. */
#define DFM_NUM_KCLASS 7
DFM_API dfm_status dfm_ctx_set_profiling(dfm_ctx* ctx, int enable);
DFM_API dfm_status dfm_ctx_kernel_times(const dfm_ctx* ctx, double* ms, int64_t* launches,
                                int64_t* voxels);

/* Kernel-family tuning of a context (no reference counterpart; defaults are
 * the tuned ones).  DFM_OPT_BRICK_MAX: pyramid levels with at most this many
 * voxels run the brick kernels, larger ones the plane-streaming kernels
 * (default 200000; 0 = never brick).  DFM_OPT_FORCE_LEGACY: 1 = run the v1
 * z-march kernels everywhere (A/B reference).  Environment variables
 * DFM_BRICK_MAX / DFM_FORCE_LEGACY set the same at context creation. */
#define DFM_OPT_BRICK_MAX 1
#define DFM_OPT_FORCE_LEGACY 2
/* DFM_OPT_PERSIST: brick levels of an LNCC registration run as one
 * persistent cooperative launch per level: 2 = bricks synchronised with
 * their 26 neighbours only (default; levels with at least two bricks per
 * SM whose bricks each get a CTA, LNCC r 1..3, sigma_grad 1.0, sigma_warp
 * 0.5, step cap <= 1.5 — others run the graph path); 3 = as 2 for brick
 * levels of any size; 1 = grid barriers between phases; 0 = one CUDA graph
 * per 8 iterations.
 * Env DFM_PERSIST. */
#define DFM_OPT_PERSIST 3
/* DFM_OPT_PDL: 1 = the loop kernels use programmatic dependent
 * launch (each kernel's CTAs are scheduled while its predecessor drains and
 * wait on griddepcontrol); 0 (default, measured no faster) = plain stream
 * order.  Env DFM_PDL. */
#define DFM_OPT_PDL 4
/* DFM_OPT_SPLIT: 1 (default) = the split update (compose once per voxel, then
 * smooth); 0 = the fused compose+smooth kernel (recomposes halo elements).
 * DFM_OPT_SPLIT_FOLD_MAX: levels below this many voxels fold the compose into
 * the smooth+Adam epilogue, larger ones run it as its own kernel (default
 * 2000000).  Both give bit-identical fields.  Env DFM_SPLIT, DFM_SPLIT_FOLD_MAX. */
#define DFM_OPT_SPLIT 5
#define DFM_OPT_SPLIT_FOLD_MAX 6
/* DFM_OPT_LARGE_MIN: pyramid levels with at least this many voxels run the
 * large-level kernel variants (fp32 two-row smooth+Adam, compose-smooth with
 * the cp.async-carried W/G gather); default 2000000.  Lowering it lets the
 * parity tests run those variants at sizes the oracle finishes quickly. */
#define DFM_OPT_LARGE_MIN 7
/* DFM_OPT_SLAB_REPL_MAX: in a z-slab registration, the coarse pyramid levels
 * with at most this many voxels run whole on every rank (no halo exchange,
 * no collective; each rank computes the same level) and only the finer levels
 * are decomposed; 0 = decompose every level.  Default 4000000. */
#define DFM_OPT_SLAB_REPL_MAX 9
/* DFM_OPT_SLAB_OVERLAP: in a z-slab registration, each stage first computes
 * the planes its neighbours need, then exchanges them on a second stream
 * while the interior planes are computed (results unchanged, bit for bit).
 * -1 (default) = on for the multi-process NCCL path, off for emulated slabs
 * (one GPU: the copies compete with the compute for HBM); 0 off; 1 on. */
#define DFM_OPT_SLAB_OVERLAP 10
/* DFM_OPT_EXACT: 1 = register_images (direct mode, SSD/LNCC) evaluates the
 * reference's arithmetic in the reference's order, one IEEE operation at a
 * time (kernels_exact.cu, compiled without FMA contraction): bit-identical
 * to the reference's result, for parity checks on chaotic inputs.  fp64
 * contexts only; unfused, so far slower than the tuned loop.  Default 0. */
#define DFM_OPT_EXACT 11
/* DFM_OPT_NARROW: 1 (default) = a plane-streaming level whose last 32-wide x
 * tile would be at most half full (e.g. 80 columns) runs the 16-wide
 * instantiation of the z-march kernels (same results); 0 = always 32-wide. */
#define DFM_OPT_NARROW 12
DFM_API dfm_status dfm_ctx_set_option(dfm_ctx* ctx, int key, int64_t value);

/* White-box read of a named device workspace buffer of the context after a
 * call (the parity tests compare the hot loop's per-kernel intermediates —
 * Adam moments, capped step, composed field, W/G — with the oracle at the
 * benchmarked size; no reference counterpart).  Copies `bytes` bytes from
 * byte `offset` of buffer `name` into `host`; DFM_E_INVALID when the buffer
 * does not exist or is smaller.  Buffers of register_images after a
 * single-scale run: "reg_u0"/"reg_u1" (ping-pong displacement, 3 planes),
 * "reg_m", "reg_nu", "reg_step", "reg_grad" (holds the composed c of the
 * split update), "reg_W", "reg_G" (3 planes), in the context precision. */
DFM_API dfm_status dfm_ctx_debug_read(dfm_ctx* ctx, const char* name, size_t offset,
                                      size_t bytes, void* host);

#ifdef __cplusplus
}
#endif

#endif /* DIFFORM_GPU_H */
