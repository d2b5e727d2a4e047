/* TEST INFRASTRUCTURE ONLY: C oracle for the multi-level F/B estimator.
 * See fgm_oracle.c for provenance (reference file:line per function). */
#ifndef FGM_ORACLE_H
#define FGM_ORACLE_H
#ifdef __cplusplus
extern "C" {
#endif

int fgmo_num_levels(int w, int h);
int fgmo_level_schedule(int w, int h, int low_res_threshold, int iters_low, int iters_high, int* out_w,
                        int* out_h, int* out_iters, int cap);
void fgmo_make_taps(int src, int dst, int* i0, int* i1, double* t);
int fgmo_solve_pixel(double alpha_i, const double intensity[3], int n, const double* nalpha, const double* nfg,
                     const double* nbg, double omega, double eps_r, int clamp, double fg_out[3],
                     double bg_out[3]);

void fgmo_resize_f64(const double* src, int sw, int sh, int nch, double* dst, int dw, int dh);
void fgmo_sweep_f64(const double* image, const double* alpha, double* fg, double* bg, int w, int h,
                    double omega, double eps_r);
int fgmo_ml_solve_f64(const double* image, const double* alpha, int w, int h, double omega, double eps_r,
                      int low_res_threshold, int iters_low, int iters_high, double* fg, double* bg,
                      double** level_fg, double** level_bg);

void fgmo_compose_f64(const double* fg, const double* bg, const double* alpha, int w, int h, int nch, double* out);
void fgmo_compose_f32(const float* fg, const float* bg, const float* alpha, int w, int h, int nch, float* out);

void fgmo_resize_f32(const float* src, int sw, int sh, int nch, float* dst, int dw, int dh);
void fgmo_sweep_f32(const float* image, const float* alpha, float* fg, float* bg, int w, int h, double omega,
                    double eps_r);
int fgmo_ml_solve_f32(const float* image, const float* alpha, int w, int h, double omega, double eps_r,
                      int low_res_threshold, int iters_low, int iters_high, float* fg, float* bg,
                      float** level_fg, float** level_bg);

#ifdef __cplusplus
}
#endif
#endif
