/*
 * fastclip_oracle.c -- CPU restatement of the FastCLIP loss step. TEST INFRASTRUCTURE ONLY:
 * the parity checker for the B200 kernels (see fastclip_oracle.h). fp64 throughout, as the
 * reference (common.hpp:8-10); arrays are row-major [rows*d] (the reference stores Eigen
 * column-major, which only changes the memory order, not the arithmetic).
 *
 * File:line citations are relative to the reference's proj/core/.
 */
#include "fastclip_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* losses.cpp:10 -- process-wide clamp counter (not thread-safe here; the oracle is serial). */
static uint64_t g_exp_clamps = 0;
static const double kExpClampMax = 60.0; /* losses.hpp:22 (kExpClampMax) */

/* losses.cpp:22-28 */
double oc_safe_exp(double x) {
  if (x > kExpClampMax) {
    ++g_exp_clamps;
    x = kExpClampMax;
  }
  return exp(x);
}
uint64_t oc_exp_clamp_count(void) { return g_exp_clamps; }   /* losses.cpp:30 */
void oc_reset_exp_clamp_count(void) { g_exp_clamps = 0; }    /* losses.cpp:31 */

/* schedules.cpp:25-31 (cosine kind; the constant kind is just `return constant`). */
double oc_gamma_cosine(long long t, long long iters_per_epoch, long long decay_epochs,
                       double gamma_min) {
  const double kPi = 3.141592653589793238462643383279502884;
  const long long epoch = t / iters_per_epoch;
  if (epoch >= decay_epochs) return gamma_min;
  const double frac = (double)epoch / (double)decay_epochs;
  return 0.5 * (1.0 + cos(kPi * frac)) * (1.0 - gamma_min) + gamma_min;
}

/* schedules.cpp:62-65 (switch_epoch < 0 means "never"). */
double oc_epsilon_at(long long epoch, double initial, double late, long long switch_epoch) {
  if (switch_epoch < 0) return initial;
  return epoch < switch_epoch ? initial : late;
}

/* schedules.hpp:55-58 -- one-way latch. */
double oc_latch_modifier(int* latched, double current_tau, double threshold, double factor) {
  if (current_tau < threshold) *latched = 1;
  return *latched ? factor : 1.0;
}

/* optimizers.cpp:65-75 */
int oc_scalar_adamw_step(double* m, double* v, int64_t* step, double theta, double grad,
                         double lr, double beta1, double beta2, double eps,
                         double weight_decay, double* theta_out) {
  if (!isfinite(grad)) return OC_ERR_NUMERIC;
  *m = beta1 * *m + (1.0 - beta1) * grad;
  *v = beta2 * *v + (1.0 - beta2) * grad * grad;
  const double c1 = 1.0 - pow(beta1, (double)(*step + 1));
  const double c2 = 1.0 - pow(beta2, (double)(*step + 1));
  ++*step;
  const double r = (*m / c1) / (sqrt(*v / c2) + eps);
  *theta_out = theta - lr * (r + weight_decay * theta);
  return OC_OK;
}

/* optimizers.cpp:77-83 -- weight decay pinned to 0, then projection onto [tau0, inf). */
int oc_temperature_step(double* m, double* v, int64_t* step, double tau, double grad,
                        double lr, double beta1, double beta2, double eps, double tau0,
                        double* tau_out) {
  double next = 0.0;
  const int rc = oc_scalar_adamw_step(m, v, step, tau, grad, lr, beta1, beta2, eps, 0.0, &next);
  if (rc != OC_OK) return rc;
  *tau_out = next < tau0 ? tau0 : next;
  return OC_OK;
}

/* losses.cpp:33-41 -- S = E1 E2^T (fp64). */
static double* similarity(int B, int d, const double* E1, const double* E2) {
  double* S = (double*)malloc(sizeof(double) * (size_t)B * (size_t)B);
  if (!S) return NULL;
  for (int i = 0; i < B; ++i) {
    const double* a = E1 + (size_t)i * d;
    for (int j = 0; j < B; ++j) {
      const double* b = E2 + (size_t)j * d;
      double acc = 0.0;
      for (int k = 0; k < d; ++k) acc += a[k] * b[k];
      S[(size_t)i * B + j] = acc;
    }
  }
  return S;
}
#define SIJ(S, B, i, j) ((S)[(size_t)(i) * (size_t)(B) + (size_t)(j)])

/* engine.cpp:11-19 (require_batch) */
static int require_batch(int B, int lo, int cnt) {
  if (B < 2) return OC_ERR_DEGENERATE;
  if (lo < 0 || cnt <= 0 || lo + cnt > B) return OC_ERR_SHAPE;
  return OC_OK;
}

/* engine.cpp:151-176 -- g1/g2 for the local anchors over G \ {i}. */
static void g_values_s(int B, const double* S, const double* t1_local, const double* t2_local,
                       int lo, int cnt, double* g1, double* g2) {
  const double inv = 1.0 / (double)(B - 1);
  for (int r = 0; r < cnt; ++r) {
    const int i = lo + r;
    const double sii = SIJ(S, B, i, i);
    double a1 = 0.0, a2 = 0.0;
    for (int j = 0; j < B; ++j) {
      if (j == i) continue;
      a1 += oc_safe_exp((SIJ(S, B, i, j) - sii) / t1_local[r]);
      a2 += oc_safe_exp((SIJ(S, B, j, i) - sii) / t2_local[r]);
    }
    g1[r] = a1 * inv;
    g2[r] = a2 * inv;
  }
}

int oc_g_values(int B, int d, const double* E1, const double* E2, const double* t1_local,
                const double* t2_local, int local_begin, int local_count, double* g1,
                double* g2) {
  int rc = require_batch(B, local_begin, local_count);
  if (rc != OC_OK) return rc;
  double* S = similarity(B, d, E1, E2);
  g_values_s(B, S, t1_local, t2_local, local_begin, local_count, g1, g2);
  free(S);
  return OC_OK;
}

/* engine.cpp:77-121 (Parts::both) -- anchor part (:93-106) + contrast part (:107-118). */
static void cotangents_s(int B, int d, const double* S, const double* E1, const double* E2,
                         const double* w1, const double* w2, const double* t1,
                         const double* t2, int lo, int cnt, double* dE1, double* dE2) {
  const double scale = 1.0 / ((double)cnt * (double)(B - 1));
  memset(dE1, 0, sizeof(double) * (size_t)cnt * d);
  memset(dE2, 0, sizeof(double) * (size_t)cnt * d);
  for (int r = 0; r < cnt; ++r) {
    const int i = lo + r;
    double* o1 = dE1 + (size_t)r * d;
    double* o2 = dE2 + (size_t)r * d;
    const double* e1i = E1 + (size_t)i * d;
    const double* e2i = E2 + (size_t)i * d;
    const double sii = SIJ(S, B, i, i);
    for (int j = 0; j < B; ++j) {
      if (j == i) continue;
      const double l1 = oc_safe_exp((SIJ(S, B, i, j) - sii) / t1[i]);
      const double l2 = oc_safe_exp((SIJ(S, B, j, i) - sii) / t2[i]);
      const double a1 = scale * w1[i] * l1 / t1[i];
      const double a2 = scale * w2[i] * l2 / t2[i];
      const double* e1j = E1 + (size_t)j * d;
      const double* e2j = E2 + (size_t)j * d;
      for (int k = 0; k < d; ++k) {
        o1[k] += a1 * (e2j[k] - e2i[k]) - a2 * e2i[k];
        o2[k] += a2 * (e1j[k] - e1i[k]) - a1 * e1i[k];
      }
    }
    for (int a = 0; a < B; ++a) {
      if (a == i) continue;
      const double saa = SIJ(S, B, a, a);
      const double l1 = oc_safe_exp((SIJ(S, B, a, i) - saa) / t1[a]);
      const double l2 = oc_safe_exp((SIJ(S, B, i, a) - saa) / t2[a]);
      const double c1 = scale * w1[a] * l1 / t1[a];
      const double c2 = scale * w2[a] * l2 / t2[a];
      const double* e1a = E1 + (size_t)a * d;
      const double* e2a = E2 + (size_t)a * d;
      for (int k = 0; k < d; ++k) o2[k] += c1 * e1a[k];
      for (int k = 0; k < d; ++k) o1[k] += c2 * e2a[k];
    }
  }
}

int oc_embedding_cotangents(int B, int d, const double* E1, const double* E2,
                            const double* w1, const double* w2, const double* t1,
                            const double* t2, int local_begin, int local_count,
                            double* dE1, double* dE2) {
  int rc = require_batch(B, local_begin, local_count);
  if (rc != OC_OK) return rc;
  double* S = similarity(B, d, E1, E2);
  cotangents_s(B, d, S, E1, E2, w1, w2, t1, t2, local_begin, local_count, dE1, dE2);
  free(S);
  return OC_OK;
}

/* engine.cpp:182-204 -- t indexed by the GLOBAL row i (:198-199). */
static void dtau_sums_s(int B, const double* S, const double* t1, const double* t2, int lo,
                        int cnt, double* dsum1, double* dsum2) {
  const double inv = 1.0 / (double)(B - 1);
  for (int r = 0; r < cnt; ++r) {
    const int i = lo + r;
    const double sii = SIJ(S, B, i, i);
    double a1 = 0.0, a2 = 0.0;
    for (int j = 0; j < B; ++j) {
      if (j == i) continue;
      const double d1 = SIJ(S, B, i, j) - sii;
      const double d2 = SIJ(S, B, j, i) - sii;
      a1 += -(d1 / (t1[i] * t1[i])) * oc_safe_exp(d1 / t1[i]);
      a2 += -(d2 / (t2[i] * t2[i])) * oc_safe_exp(d2 / t2[i]);
    }
    dsum1[r] = a1 * inv;
    dsum2[r] = a2 * inv;
  }
}

int oc_dtau_sums(int B, int d, const double* E1, const double* E2, const double* t1,
                 const double* t2, int local_begin, int local_count, double* dsum1,
                 double* dsum2) {
  int rc = require_batch(B, local_begin, local_count);
  if (rc != OC_OK) return rc;
  double* S = similarity(B, d, E1, E2);
  dtau_sums_s(B, S, t1, t2, local_begin, local_count, dsum1, dsum2);
  free(S);
  return OC_OK;
}

/* losses.cpp:103-114 (g_full) */
static void g_full_s(int B, const double* S, int i, double tau1, double tau2, double* g1,
                     double* g2) {
  double a1 = 0.0, a2 = 0.0;
  const double sii = SIJ(S, B, i, i);
  for (int j = 0; j < B; ++j) {
    if (j == i) continue;
    a1 += oc_safe_exp((SIJ(S, B, i, j) - sii) / tau1);
    a2 += oc_safe_exp((SIJ(S, B, j, i) - sii) / tau2);
  }
  const double m = (double)(B - 1);
  *g1 = a1 / m;
  *g2 = a2 / m;
}

/* losses.cpp:126-138 */
static double eval_gcl_s(int B, const double* S, double tau, double eps) {
  double acc = 0.0;
  for (int i = 0; i < B; ++i) {
    double g1, g2;
    g_full_s(B, S, i, tau, tau, &g1, &g2);
    acc += log(eps + g1) + log(eps + g2);
  }
  return tau * acc / (double)B;
}
double oc_eval_gcl(int B, int d, const double* E1, const double* E2, double tau, double eps) {
  double* S = similarity(B, d, E1, E2);
  const double v = eval_gcl_s(B, S, tau, eps);
  free(S);
  return v;
}

/* losses.cpp:140-159 */
static double eval_rgcl_s(int B, const double* S, const double* tau1, const double* tau2,
                          double eps, double rho) {
  double acc = 0.0;
  for (int i = 0; i < B; ++i) {
    double g1, g2;
    g_full_s(B, S, i, tau1[i], tau2[i], &g1, &g2);
    acc += tau1[i] * (log(eps + g1) + rho);
    acc += tau2[i] * (log(eps + g2) + rho);
  }
  return acc / (double)B;
}
double oc_eval_rgcl(int B, int d, const double* E1, const double* E2, const double* tau1,
                    const double* tau2, double eps, double rho) {
  double* S = similarity(B, d, E1, E2);
  const double v = eval_rgcl_s(B, S, tau1, tau2, eps, rho);
  free(S);
  return v;
}

/* losses.cpp:168-180 */
static double eval_mbcl_s(int B, const double* S, double tau) {
  const double c = 1.0 / (double)(B - 1);
  double acc = 0.0;
  for (int i = 0; i < B; ++i) {
    double g1, g2;
    g_full_s(B, S, i, tau, tau, &g1, &g2);
    acc += log(c + g1) + log(c + g2);
  }
  return acc / (double)B;
}
double oc_eval_mbcl(int B, int d, const double* E1, const double* E2, double tau) {
  double* S = similarity(B, d, E1, E2);
  const double v = eval_mbcl_s(B, S, tau);
  free(S);
  return v;
}

static int uses_u(int v) { return v != OC_OPENCLIP_MBCL; }                  /* trainer.cpp:39 */
static int individual(int v) { return v == OC_ISOGCLR || v == OC_FASTCLIP_V2; } /* :41-43 */
static int scheme_global_v0(int v) { return v == OC_OPENCLIP_MBCL || v == OC_FASTCLIP_V0; } /* :45-56 */
static int scheme_constant(int v) { return v == OC_SOGCLR || v == OC_FASTCLIP_V1; }

/*
 * trainer.cpp:427-589 for workers k = 0..K-1 with the FastCLIP (all-gather) reduction.
 * Phase 1 (per worker, up to the u-gather rendezvous at :464): g at tau^t, EMA update of the
 * owned u entries, snapshot. Phase 2 (after the gathers): weights, cotangents, tau gradients.
 * The serial two-phase replay is exactly what the fabric's barriers enforce.
 */
int oc_step(const oc_config* cfg, oc_state* st, int K, int B, int d, const double* E1,
            const double* E2, const int32_t* ids, double gamma, double eps, oc_step_out* out) {
  if (K < 1 || B % K != 0) return OC_ERR_SHAPE;
  if (B < 2) return OC_ERR_DEGENERATE;
  const int Bl = B / K;
  const int v = cfg->variant;
  const int track_u = uses_u(v);
  const int indiv = individual(v);
  if (eps < 0.0) return OC_ERR_DOMAIN;                     /* engine.cpp:29 */
  if (!indiv && !(st->tau > 0.0)) return OC_ERR_DOMAIN;    /* engine.cpp:39 */
  if (track_u && (!(gamma > 0.0) || gamma > 1.0)) return OC_ERR_DOMAIN; /* state.cpp:50 */
  for (int i = 0; i < B; ++i)
    if (ids[i] < 0 || (int64_t)ids[i] >= cfg->n_train) return OC_ERR_SHAPE; /* state.cpp:46 */

  double* S = similarity(B, d, E1, E2);
  double* w1 = (double*)malloc(sizeof(double) * B);
  double* w2 = (double*)malloc(sizeof(double) * B);
  double* tt1 = (double*)malloc(sizeof(double) * B);
  double* tt2 = (double*)malloc(sizeof(double) * B);
  double* ds1 = (double*)malloc(sizeof(double) * Bl);
  double* ds2 = (double*)malloc(sizeof(double) * Bl);
  int rc = OC_OK;

  /* ---- phase 1: tau^t snapshot (:428-434), g (:436), u update + snapshot (:439-445) ---- */
  out->clamps_g = 0;
  for (int k = 0; k < K; ++k) {
    for (int r = 0; r < Bl; ++r) {
      const int i = k * Bl + r;
      out->t1[i] = indiv ? st->tau1[ids[i]] : st->tau;
      out->t2[i] = indiv ? st->tau2[ids[i]] : st->tau;
    }
    const uint64_t c0 = g_exp_clamps;
    g_values_s(B, S, out->t1 + k * Bl, out->t2 + k * Bl, k * Bl, Bl, out->g1 + k * Bl,
               out->g2 + k * Bl);
    out->clamps_g += g_exp_clamps - c0;
    if (track_u) {
      for (int r = 0; r < Bl; ++r) {
        const int i = k * Bl + r;
        const double g1 = out->g1[i], g2 = out->g2[i];
        if (g1 < 0.0 || g2 < 0.0) { rc = OC_ERR_DOMAIN; goto done; } /* state.cpp:51 */
        const int p = ids[i];
        st->u1[p] = (1.0 - gamma) * st->u1[p] + gamma * g1;          /* state.cpp:52 */
        st->u2[p] = (1.0 - gamma) * st->u2[p] + gamma * g2;          /* state.cpp:53 */
      }
      for (int r = 0; r < Bl; ++r) {                                  /* state.cpp:57-71 */
        const int i = k * Bl + r;
        out->u1[i] = st->u1[ids[i]];
        out->u2[i] = st->u2[ids[i]];
      }
    }
  }

  /* ---- weights over the whole global batch (:449-491) ---- */
  if (v == OC_OPENCLIP_MBCL) {
    /* :451-457 -- g over ALL anchors at tau, weights_mbcl (engine.cpp:65-75), u := g */
    double* ta = (double*)malloc(sizeof(double) * B);
    for (int i = 0; i < B; ++i) ta[i] = st->tau;
    g_values_s(B, S, ta, ta, 0, B, out->u1, out->u2);
    free(ta);
    const double c = 1.0 / (double)(B - 1);
    for (int i = 0; i < B; ++i) {
      tt1[i] = st->tau; tt2[i] = st->tau;
      w1[i] = 1.0 / (c + out->u1[i]);
      w2[i] = 1.0 / (c + out->u2[i]);
    }
  } else if (indiv) {
    /* engine.cpp:52-63 -- w = (1/(eps+u)) * tau_i, t = tau_i (u-gather :464, tau-gather :479) */
    for (int i = 0; i < B; ++i) {
      tt1[i] = out->t1[i]; tt2[i] = out->t2[i];
      w1[i] = (1.0 / (eps + out->u1[i])) * out->t1[i];
      w2[i] = (1.0 / (eps + out->u2[i])) * out->t2[i];
    }
  } else {
    /* engine.cpp:37-50 -- w = 1/(eps+u), times tau when scaled */
    for (int i = 0; i < B; ++i) {
      tt1[i] = st->tau; tt2[i] = st->tau;
      w1[i] = 1.0 / (eps + out->u1[i]);
      w2[i] = 1.0 / (eps + out->u2[i]);
      if (cfg->scale_by_tau) { w1[i] *= st->tau; w2[i] *= st->tau; }
    }
  }

  /* ---- phase 2 per worker: cotangents (:522-524), tau gradients (:557-589) ---- */
  for (int k = 0; k < K; ++k) {
    cotangents_s(B, d, S, E1, E2, w1, w2, tt1, tt2, k * Bl, Bl, out->dE1 + (size_t)k * Bl * d,
                 out->dE2 + (size_t)k * Bl * d);
    out->gtau_local[k] = 0.0;
    if (scheme_constant(v)) continue;
    if (indiv) {
      /* engine.cpp:240-259 with dataset_size = n_train */
      if (cfg->n_train < 2) { rc = OC_ERR_DEGENERATE; goto done; }
      dtau_sums_s(B, S, tt1, tt2, k * Bl, Bl, ds1, ds2);
      const double inv_n = 1.0 / (double)cfg->n_train;
      for (int r = 0; r < Bl; ++r) {
        const int i = k * Bl + r;
        out->gtau1[i] = inv_n * (log(eps + out->u1[i]) + cfg->rho +
                                 tt1[i] * ds1[r] / (eps + out->u1[i]));
        out->gtau2[i] = inv_n * (log(eps + out->u2[i]) + cfg->rho +
                                 tt2[i] * ds2[r] / (eps + out->u2[i]));
      }
      continue;
    }
    /* engine.cpp:208-224 (v0), :226-238 (v3), :261-266 (mbcl: eps := 1/(B-1), u := g) */
    const double e = (v == OC_OPENCLIP_MBCL) ? 1.0 / (double)(B - 1) : eps;
    dtau_sums_s(B, S, tt1, tt2, k * Bl, Bl, ds1, ds2);
    double acc = 0.0;
    for (int r = 0; r < Bl; ++r) {
      const int i = k * Bl + r;
      acc += ds1[r] / (e + out->u1[i]) + ds2[r] / (e + out->u2[i]);
    }
    const double unscaled = acc / (double)Bl;
    if (v == OC_FASTCLIP_V3) {
      double logs = 0.0;
      for (int r = 0; r < Bl; ++r) {
        const int i = k * Bl + r;
        logs += log(eps + out->u1[i]) + log(eps + out->u2[i]);
      }
      logs /= (double)Bl;
      out->gtau_local[k] = logs + 2.0 * cfg->rho + st->tau * unscaled;
    } else {
      out->gtau_local[k] = unscaled;
    }
  }

  /* ---- exact loss at tau^t (the reference evaluates it per epoch, trainer.cpp:620) ---- */
  if (v == OC_OPENCLIP_MBCL) out->loss = eval_mbcl_s(B, S, st->tau);
  else if (indiv) out->loss = eval_rgcl_s(B, S, out->t1, out->t2, eps, cfg->rho);
  else if (v == OC_FASTCLIP_V3) out->loss = eval_gcl_s(B, S, st->tau, eps) + 2.0 * cfg->rho * st->tau;
  else out->loss = eval_gcl_s(B, S, st->tau, eps);

  /* ---- temperature update (:557-589) ---- */
  out->gtau = 0.0;
  out->tau_new = st->tau;
  if (indiv) {
    /* state.cpp:124-131 per owned index; every id of the global batch is owned by someone */
    for (int i = 0; i < B; ++i) {
      const int p = ids[i];
      double nt;
      rc = oc_temperature_step(&st->m1[p], &st->v1[p], &st->s1[p], st->tau1[p], out->gtau1[i],
                               cfg->tau_lr, cfg->beta1, cfg->beta2, cfg->adam_eps, cfg->tau0, &nt);
      if (rc != OC_OK) goto done;
      st->tau1[p] = nt;
      rc = oc_temperature_step(&st->m2[p], &st->v2[p], &st->s2[p], st->tau2[p], out->gtau2[i],
                               cfg->tau_lr, cfg->beta1, cfg->beta2, cfg->adam_eps, cfg->tau0, &nt);
      if (rc != OC_OK) goto done;
      st->tau2[p] = nt;
    }
  } else if (!scheme_constant(v)) {
    /* fabric.cpp:73-83 reduce_mean: ascending-order sum times 1/K */
    double sum = 0.0;
    for (int k = 0; k < K; ++k) sum += out->gtau_local[k];
    out->gtau = sum * (1.0 / (double)K);
    double lr = cfg->tau_lr;
    if (cfg->lr_decay_enabled)
      lr *= oc_latch_modifier(&st->latched, st->tau, cfg->lr_decay_threshold,
                              cfg->lr_decay_factor);
    double nt;
    rc = oc_temperature_step(&st->tau_m, &st->tau_v, &st->tau_step, st->tau, out->gtau, lr,
                             cfg->beta1, cfg->beta2, cfg->adam_eps, cfg->tau0, &nt);
    if (rc != OC_OK) goto done;
    st->tau = nt;
    out->tau_new = nt;
  }

done:
  free(S); free(w1); free(w2); free(tt1); free(tt2); free(ds1); free(ds2);
  return rc;
}
