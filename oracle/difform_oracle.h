/*
 * oracle/difform_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C, fp64, single-threaded restatement of the reference's hot path
 * (difform, /root/reference/proj/src).  It is the CHECKER for the CUDA path:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it.  The product library never links it and has no CPU fallback.
 *
 * Pinning: tests/test_oracle.py checks every function here against golden
 * vectors produced by the UNMODIFIED reference compiled from its own sources
 * (oracle/Makefile `ref` target -> oracle/_ref/libdifform_ref.so; generator
 * tests/golden/make_golden.py).  Bit-identical is expected and tested:
 * operation order follows the reference (no FMA contraction at -O2 x86-64,
 * the 4096-element block-ordered sum of parallel.cpp:153-169).
 *
 * Conventions follow include/difform_gpu.h: host AoS doubles, dfm_grid,
 * return 0 ok / 1 invalid argument / 2 numerical failure.
 */
#ifndef DIFFORM_ORACLE_H
#define DIFFORM_ORACLE_H

#include "../include/difform_gpu.h"

#ifdef __cplusplus
extern "C" {
#endif

size_t orc_last_error(char* buf, size_t cap);
int orc_validate_grid(const dfm_grid* g);
int orc_downsample_grid(const dfm_grid* g, const double factor[3], dfm_grid* out);
int orc_downsample_image(const dfm_grid* g, const double* img, const double factor[3],
                         dfm_grid* out_grid, double* out);
int orc_sample_linear_points(const dfm_grid* g, const double* img, int64_t npts,
                             const double* pts, double* values, double* grads);
int orc_warp_image(const dfm_grid* g, const double* img, const double* phi, double* out);
int orc_warp_labels(const dfm_grid* g, const int32_t* labels, const double* phi,
                    int32_t* out);
int orc_compose(const dfm_grid* g, const double* phi, const double* psi, double* out);
int orc_jacobian_det(const dfm_grid* g, const double* phi, double* out);
int orc_gaussian_smooth(const dfm_grid* g, const double* img, const double sigma[3],
                        double* out);
int orc_gaussian_smooth_field(const dfm_grid* g, const double* f, const double sigma[3],
                              double* out);
int orc_upsample_field(const dfm_grid* g, const double* phi, const dfm_grid* ng, double* out);
int orc_resample_field_linear(const dfm_grid* g, const double* f, const dfm_grid* ng,
                              double* out);
int orc_resample_displacement(const dfm_grid* g, const double* phi, const dfm_grid* ng,
                              double* out);
int orc_ssd_eval(const dfm_grid* fg, const double* fixed, const dfm_grid* mg,
                 const double* moving, const double* phi, double* value, double* grad);
int orc_lncc_eval(const dfm_grid* fg, const double* fixed, const dfm_grid* mg,
                  const double* moving, const double* phi, int r, double* value, double* grad);
int orc_dice_eval(const dfm_grid* fg, const double* fixed, const dfm_grid* mg,
                  const double* moving, const double* phi, double* value, double* grad);
int orc_adam_step(const dfm_grid* g, double* m, double* nu, int64_t* t, double b1, double b2,
                  double eps, const double* v, double* dir);
int orc_upsample_state(const dfm_grid* g, const double* m, const double* nu,
                       const dfm_grid* ng, double* m_out, double* nu_out);
int orc_eulerian_direction(const dfm_grid* g, const double* grad, const double* phi,
                           int use_jac, double* out);
int orc_apply_update(const dfm_grid* g, const double* phi, const double* v, double eta,
                     double sigma_warp, double cap, double* out);
int orc_singularity_fraction(const dfm_grid* g, const double* phi, double* frac);
int orc_affine_to_field(const dfm_grid* g, const double A[9], const double t[3], double* out);
int orc_affine_param_gradient(const dfm_grid* g, const double* fixed, const double* moving,
                              int loss, const double A[9], const double t[3], const double S[3],
                              int lncc_radius, double* value, double dA[9], double dt[3]);
int orc_affine_register(const dfm_grid* g, const double* fixed, const double* moving, int loss,
                        const double* scales, const int32_t* iters, int32_t nscales, double eta,
                        int lncc_radius, dfm_affine_result* out);
int orc_exp_map(const dfm_grid* g, const double* v, int M, double* out);
int orc_svf_pullback(const dfm_grid* g, const double* v, const double* grad_phi, int M,
                     double* out);
int orc_register(const dfm_grid* g, const double* fixed, const double* moving,
                 const dfm_config* cfg, const double* scales, const int32_t* iters,
                 int32_t nscales, const dfm_init* init, double* out_field,
                 dfm_iter_record* records, int64_t max_records, dfm_runlog* log);
int orc_overlap_report(const dfm_grid* gw, const int32_t* warped, const dfm_grid* gf,
                       const int32_t* fixed, dfm_overlap_summary* rep,
                       dfm_region_overlap* regions, int64_t cap);
int orc_landmark_error(const dfm_grid* fg, const dfm_grid* mg, const dfm_grid* pg,
                       const double* phi, int64_t n, const double* fixed_mm,
                       const double* moving_mm, double* dist, double* mean, double* mx);
int orc_sweep(const dfm_sweep_pair* pairs, int npairs, const dfm_config* base,
              const double* scales, const int32_t* iters, int32_t nscales, const double* etas,
              int n_eta, const double* sws, int n_sw, const double* sgs, int n_sg, int metric,
              dfm_sweep_row* rows);
int orc_overlap_dice(const dfm_grid* g, const int32_t* warped, const int32_t* fixed,
                     double* mo_mean, double* mo_klein);

#ifdef __cplusplus
}
#endif

#endif
