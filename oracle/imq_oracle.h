/* imq_oracle.h -- CPU restatement of the reference fast IMQ path.
 * TEST INFRASTRUCTURE ONLY (see imq_oracle.c header). Returns 0 on success,
 * -1 on error with ora_last_error() describing it. */
#ifndef IMQ_ORACLE_H
#define IMQ_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
const char* ora_last_error(void);
int ora_random_vector(int64_t n, uint64_t seed, double* out);
int ora_halton2d(int64_t n, double* xy);
double ora_rel_err_inf(const double* test, const double* ref, int64_t n);
void ora_legendre_table(int M, double x, double sin_theta, double* out);
void ora_coeff_d_table(int M, double* out);
int ora_auto_level(int N, int M);
double ora_cost_upper_bound(int N, int M, int L);
int ora_bounding_square(const double* xy, int64_t n, double* sq3);
int ora_block_ids(const double* xy, int64_t n, int level, int32_t* out);
int ora_interaction_list(int level, int i, int j, int32_t* out);
int ora_resolved_levels(int64_t n, int M, int L);
int ora_fast_matvec(const double* xy, int64_t n, double t, int M, int L, const double* u,
                    double* b);
int ora_fast_matvec_rows(const double* xy, int64_t n, double t, int M, int L, const double* u,
                         const int64_t* rows, int64_t nrows, double* b_rows);
int ora_block_moments(const double* xy, int64_t n, double t, int M, int L, const double* u,
                      int level, int block, double* v, double* w);
int ora_dense_rows(const double* xy, int64_t n, double t, const double* u, const int64_t* rows,
                   int64_t nrows, double* out);
int ora_dense_matvec(const double* xy, int64_t n, double t, const double* u, double* b);
int ora_iterative_solve(const double* xy, int64_t n, double t, int M, int L, const double* f,
                        double tol, int max_iter, int restart, double* c_out, int* iterations,
                        double* final_rel, int* converged, double* cycle_res, int max_cycles,
                        int* n_cycles);
int ora_evaluate_interpolant(const double* cxy, const double* c, int64_t n, double t,
                             const double* qxy, int64_t nq, double* out);
#ifdef __cplusplus
}
#endif
#endif
