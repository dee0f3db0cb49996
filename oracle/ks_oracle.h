/* ORACLE -- TEST INFRASTRUCTURE ONLY (see ks_oracle.c).  Shares nothing with
 * the CUDA path's include/ks.h. */
#ifndef KS_ORACLE_H
#define KS_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
int oracle_whiten(int64_t N, int n, int m_max, const int32_t *m,
                  const double *F, int64_t sF, const double *H, int64_t sH,
                  const double *c, int64_t sc, const double *o, int64_t so,
                  const double *K, int64_t sK, const double *L, int64_t sL,
                  double *C, double *y, double *B, double *D, double *e,
                  int64_t *bad_step, int *bad_kind);
int oracle_factor(int64_t N, int n, int m_max, const int32_t *m,
                  const double *C, const double *y, const double *B, const double *D,
                  const double *e, double *Rd, double *Ro, double *z, int64_t *bad_step);
int oracle_solve(int64_t N, int n, const double *Rd, const double *Ro, const double *z, double *x);
int oracle_selinv(int64_t N, int n, const double *Rd, const double *Ro, double *S, double *Scross);
int oracle_smooth(int64_t N, int n, int m_max, const int32_t *m,
                  const double *F, int64_t sF, const double *H, int64_t sH,
                  const double *c, int64_t sc, const double *o, int64_t so,
                  const double *K, int64_t sK, const double *L, int64_t sL,
                  double *x, double *S, int64_t *bad_step, int *bad_kind);
#ifdef __cplusplus
}
#endif
#endif
