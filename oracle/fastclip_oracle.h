/*
 * fastclip_oracle.h -- CPU restatement of the FastCLIP loss step (TEST INFRASTRUCTURE ONLY).
 *
 * This is the parity checker for the B200 path, never the product: only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may load it.
 * Every function restates the reference algorithm in plain C (fp64, row-major arrays) and
 * cites the reference file:line it follows (paths relative to proj/core of the reference).
 *
 * Parity pinning: this restatement is checked against (a) the SPEC.md known answers and
 * (b) golden vectors produced by the reference's OWN translation units (engine.cpp,
 * losses.cpp, state.cpp, optimizers.cpp, schedules.cpp, fabric.cpp) compiled against a
 * local Eigen-subset shim (oracle/ref_shim, oracle/Makefile -> oracle/_ref/).
 */
#ifndef FASTCLIP_ORACLE_H
#define FASTCLIP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Variant ids in the reference's enum order (trainer.hpp:145-153). */
enum {
  OC_OPENCLIP_MBCL = 0,
  OC_SOGCLR = 1,
  OC_ISOGCLR = 2,
  OC_FASTCLIP_V0 = 3,
  OC_FASTCLIP_V1 = 4,
  OC_FASTCLIP_V2 = 5,
  OC_FASTCLIP_V3 = 6
};

/* Status codes: one per exception class of errors.hpp:10-60 (+ std::domain_error). */
enum {
  OC_OK = 0,
  OC_ERR_CONFIG = 1,
  OC_ERR_SHAPE = 2,
  OC_ERR_DEGENERATE = 3,
  OC_ERR_DOMAIN = 4,
  OC_ERR_OWNERSHIP = 5,
  OC_ERR_STALENESS = 6,
  OC_ERR_NUMERIC = 9
};

/* Resolved temperature / optimizer settings (trainer.cpp:139-194, state.hpp:71-89,
 * optimizers.hpp:10-15). */
typedef struct {
  int variant;
  int64_t n_train;          /* N: table size and the v2 1/N prefactor (trainer.cpp:580-582) */
  double tau0;              /* projection floor */
  double rho;
  double tau_lr;
  double beta1, beta2, adam_eps;
  int lr_decay_enabled;     /* TauLrLatch in use (v3 default) */
  double lr_decay_threshold;
  double lr_decay_factor;
  int scale_by_tau;         /* w = tau/(eps+u) if 1, 1/(eps+u) if 0 (engine.cpp:37-50) */
} oc_config;

/* Run state that persists across steps (tables are dataset-sized, fp64). */
typedef struct {
  double* u1; double* u2;                 /* UTable (state.hpp:37-69), u0 = 0 */
  double* tau1; double* tau2;             /* IndividualTemp (v2 only, else NULL) */
  double* m1; double* v1; int64_t* s1;    /* ScalarAdam track 1 (AoS in the reference) */
  double* m2; double* v2; int64_t* s2;    /* ScalarAdam track 2 */
  double tau;                             /* global tau (Replica::tau) */
  double tau_m, tau_v; int64_t tau_step;  /* Replica::tau_adam */
  int latched;                            /* Replica::latch.latched */
} oc_state;

/* Per-step outputs; arrays are global-batch sized, rank k's rows at [k*Bl, (k+1)*Bl). */
typedef struct {
  double* dE1; double* dE2;   /* [B*d] embedding cotangents (engine.cpp:77-121) */
  double* g1; double* g2;     /* [B] inner means at tau^t (engine.cpp:151-176) */
  double* u1; double* u2;     /* [B] u^{t+1} snapshot (state.cpp:57-71); g for mbcl */
  double* t1; double* t2;     /* [B] temperatures tau^t used by the step */
  double* gtau1; double* gtau2; /* [B] v2 per-index tau gradients (engine.cpp:240-259) */
  double* gtau_local;         /* [K] per-worker G_tau before the mean all-reduce */
  double gtau;                /* all_reduce_mean of gtau_local (fabric.cpp:210-212) */
  double tau_new;             /* global tau after temperature_step */
  double loss;                /* exact batch loss at tau^t (losses.cpp:126-180) */
  uint64_t clamps_g;          /* safe_exp clamps inside the local g_values calls */
} oc_step_out;

/* ---- scalar building blocks ---- */
double oc_safe_exp(double x);                 /* losses.cpp:22-28 */
uint64_t oc_exp_clamp_count(void);            /* losses.cpp:30 */
void oc_reset_exp_clamp_count(void);          /* losses.cpp:31 */
double oc_gamma_cosine(long long t, long long iters_per_epoch, long long decay_epochs,
                       double gamma_min);     /* schedules.cpp:25-31 */
double oc_epsilon_at(long long epoch, double initial, double late,
                     long long switch_epoch); /* schedules.cpp:62-65 */
double oc_latch_modifier(int* latched, double current_tau, double threshold,
                         double factor);      /* schedules.hpp:55-58 */
int oc_scalar_adamw_step(double* m, double* v, int64_t* step, double theta, double grad,
                         double lr, double beta1, double beta2, double eps,
                         double weight_decay, double* theta_out); /* optimizers.cpp:65-75 */
int oc_temperature_step(double* m, double* v, int64_t* step, double tau, double grad,
                        double lr, double beta1, double beta2, double eps, double tau0,
                        double* tau_out);     /* optimizers.cpp:77-83 */

/* ---- batch building blocks (E row-major [B*d] doubles) ---- */
int oc_g_values(int B, int d, const double* E1, const double* E2, const double* t1_local,
                const double* t2_local, int local_begin, int local_count, double* g1,
                double* g2);                  /* engine.cpp:151-176 */
int oc_embedding_cotangents(int B, int d, const double* E1, const double* E2,
                            const double* w1, const double* w2, const double* t1,
                            const double* t2, int local_begin, int local_count,
                            double* dE1, double* dE2); /* engine.cpp:77-121 */
int oc_dtau_sums(int B, int d, const double* E1, const double* E2, const double* t1,
                 const double* t2, int local_begin, int local_count, double* dsum1,
                 double* dsum2);              /* engine.cpp:182-204 */
double oc_eval_gcl(int B, int d, const double* E1, const double* E2, double tau,
                   double eps);               /* losses.cpp:126-138 */
double oc_eval_rgcl(int B, int d, const double* E1, const double* E2, const double* tau1,
                    const double* tau2, double eps, double rho); /* losses.cpp:140-159 */
double oc_eval_mbcl(int B, int d, const double* E1, const double* E2,
                    double tau);              /* losses.cpp:168-180 */

/* ---- the hot-path step: trainer.cpp:427-589 replayed for all K workers ----
 * ids: [B] distinct table indices of the global batch (worker k owns ids[k*Bl .. ]).
 * gamma, eps: the step's gamma_t (schedules.cpp:25-31) and eps_t (schedules.cpp:62-65).
 * state is updated in place (u table, tau tables / Adam states, global tau, latch). */
int oc_step(const oc_config* cfg, oc_state* st, int K, int B, int d, const double* E1,
            const double* E2, const int32_t* ids, double gamma, double eps, oc_step_out* out);

#ifdef __cplusplus
}
#endif
#endif
