// ref_driver.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A C-ABI harness around the reference's OWN hot-path code (engine.cpp, losses.cpp,
// state.cpp, optimizers.cpp, schedules.cpp, fabric.cpp, compiled unmodified from
// /root/reference against oracle/ref_shim). It replays the per-worker loss step of
// Trainer::run (trainer.cpp:427-589) with the reference's own objects -- UTable,
// IndividualTemp, ScalarAdam, TauLrLatch and a K-thread dist::Fabric -- so the golden
// vectors and the CPU baseline come from the reference implementation itself.
// The encoder/model side of the step (trainer.cpp:412-425, 539-553) is out of scope: the
// gathered embeddings are given directly.
#include <cstring>
#include <memory>
#include <span>
#include <sstream>
#include <stdexcept>
#include <vector>

#include "fastclip/engine.hpp"
#include "fastclip/fabric.hpp"
#include "fastclip/losses.hpp"
#include "fastclip/optimizers.hpp"
#include "fastclip/schedules.hpp"
#include "fastclip/state.hpp"
#include "fastclip_oracle.h"

using namespace fastclip;

namespace {

int status_of(const std::exception_ptr& e) {
  try {
    std::rethrow_exception(e);
  } catch (const ConfigError&) {
    return OC_ERR_CONFIG;
  } catch (const ShapeError&) {
    return OC_ERR_SHAPE;
  } catch (const DegenerateBatchError&) {
    return OC_ERR_DEGENERATE;
  } catch (const OwnershipViolation&) {
    return OC_ERR_OWNERSHIP;
  } catch (const StalenessError&) {
    return OC_ERR_STALENESS;
  } catch (const NumericError&) {
    return OC_ERR_NUMERIC;
  } catch (const std::domain_error&) {
    return OC_ERR_DOMAIN;
  } catch (...) {
    return 99;
  }
}

Matrix from_rows(const double* p, int rows, int cols) {
  Matrix m(rows, cols);
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) m(r, c) = p[static_cast<size_t>(r) * cols + c];
  return m;
}

void to_rows(const Matrix& m, double* p) {
  for (Eigen::Index r = 0; r < m.rows(); ++r)
    for (Eigen::Index c = 0; c < m.cols(); ++c) p[r * m.cols() + c] = m(r, c);
}

Vector from_array(const double* p, int n) {
  Vector v(n);
  for (int i = 0; i < n; ++i) v[i] = p[i];
  return v;
}

bool individual(int v) { return v == OC_ISOGCLR || v == OC_FASTCLIP_V2; }

struct Replica {  // per-worker replicated scalar state (trainer.cpp:245-254)
  double tau = 0.0;
  opt::ScalarAdam tau_adam;
  sched::TauLrLatch latch;
};

struct RefCtx {
  oc_config cfg{};
  opt::AdamConfig adam;
  std::unique_ptr<state::UTable> utable;
  state::IndividualTemp itemp;
  Replica rep;
  long long step = 0;
};

}  // namespace

extern "C" {

void* ref_create(const oc_config* cfg) {
  auto* c = new RefCtx;
  c->cfg = *cfg;
  c->adam.beta1 = cfg->beta1;
  c->adam.beta2 = cfg->beta2;
  c->adam.eps = cfg->adam_eps;
  c->adam.weight_decay = 0.0;
  c->utable = std::make_unique<state::UTable>(static_cast<int>(cfg->n_train));
  c->rep.latch.threshold = cfg->lr_decay_threshold;
  c->rep.latch.factor = cfg->lr_decay_factor;
  return c;
}

void ref_destroy(void* h) { delete static_cast<RefCtx*>(h); }

// Loads u tables, (v2) temperatures + sparse Adam slots in the reference's own binary
// format (state.cpp:133-162), and the replica's global tau state.
int ref_set_state(void* h, const oc_state* st) {
  auto* c = static_cast<RefCtx*>(h);
  const int n = static_cast<int>(c->cfg.n_train);
  c->utable->load(from_array(st->u1, n), from_array(st->u2, n));
  if (individual(c->cfg.variant)) {
    std::stringstream ss;
    auto put = [&](const void* p, size_t b) { ss.write(static_cast<const char*>(p), b); };
    const std::int64_t nn = n;
    put(&nn, 8); put(st->tau1, 8u * n);
    put(&nn, 8); put(st->tau2, 8u * n);
    put(&c->cfg.tau0, 8);
    for (int i = 0; i < n; ++i) { put(&st->m1[i], 8); put(&st->v1[i], 8); long long s = st->s1[i]; put(&s, 8); }
    for (int i = 0; i < n; ++i) { put(&st->m2[i], 8); put(&st->v2[i], 8); long long s = st->s2[i]; put(&s, 8); }
    c->itemp = state::IndividualTemp::read(ss);
  }
  c->rep.tau = st->tau;
  c->rep.tau_adam.m = st->tau_m;
  c->rep.tau_adam.v = st->tau_v;
  c->rep.tau_adam.step = st->tau_step;
  c->rep.latch.latched = st->latched != 0;
  return OC_OK;
}

int ref_get_state(void* h, oc_state* st) {
  auto* c = static_cast<RefCtx*>(h);
  const int n = static_cast<int>(c->cfg.n_train);
  std::memcpy(st->u1, c->utable->u1().data(), 8u * n);
  std::memcpy(st->u2, c->utable->u2().data(), 8u * n);
  if (individual(c->cfg.variant)) {
    std::memcpy(st->tau1, c->itemp.tau1().data(), 8u * n);
    std::memcpy(st->tau2, c->itemp.tau2().data(), 8u * n);
    for (int i = 0; i < n; ++i) {
      st->m1[i] = c->itemp.adam1()[i].m; st->v1[i] = c->itemp.adam1()[i].v; st->s1[i] = c->itemp.adam1()[i].step;
      st->m2[i] = c->itemp.adam2()[i].m; st->v2[i] = c->itemp.adam2()[i].v; st->s2[i] = c->itemp.adam2()[i].step;
    }
  }
  st->tau = c->rep.tau;
  st->tau_m = c->rep.tau_adam.m;
  st->tau_v = c->rep.tau_adam.v;
  st->tau_step = c->rep.tau_adam.step;
  st->latched = c->rep.latch.latched ? 1 : 0;
  return OC_OK;
}

// One loss step for K workers (K std::threads meeting in the reference's Fabric).
// local_limit > 0 restricts every worker's anchor loops to its first local_limit anchors
// (the bounded CPU-baseline sample; S products stay full size as in the reference).
int ref_step_ex(void* h, int K, int B, int d, const double* E1, const double* E2,
                const int32_t* ids, double gamma, double eps, oc_step_out* out,
                int local_limit, int want_loss) {
  auto* c = static_cast<RefCtx*>(h);
  try {
    if (K < 1 || B % K != 0) throw ShapeError("ref_step: K must divide B");
    const int Bl = B / K;
    const int La = (local_limit > 0 && local_limit < Bl) ? local_limit : Bl;
    const int v = c->cfg.variant;
    const bool track_u = v != OC_OPENCLIP_MBCL;
    const bool indiv = individual(v);
    const long long t = c->step++;
    const Matrix e1g = from_rows(E1, B, d);
    const Matrix e2g = from_rows(E2, B, d);

    // Epoch-style ownership claim for this step's ids (trainer.cpp:396-400).
    for (int k = 0; k < K; ++k)
      for (int r = 0; r < Bl; ++r) c->utable->owners().assign(ids[k * Bl + r], k);

    // Clamp count of the local g evaluations, measured serially (the process-wide
    // counter, losses.cpp:10, cannot separate concurrent workers).
    out->clamps_g = 0;
    if (want_loss) {
      for (int k = 0; k < K; ++k) {
        Vector tl1(La), tl2(La), ga, gb;
        for (int r = 0; r < La; ++r) {
          const int id = ids[k * Bl + r];
          tl1[r] = indiv ? c->itemp.tau1()[id] : c->rep.tau;
          tl2[r] = indiv ? c->itemp.tau2()[id] : c->rep.tau;
        }
        const auto c0 = losses::exp_clamp_count();
        engine::g_values(e1g, e2g, tl1, tl2, k * Bl, La, ga, gb);
        out->clamps_g += losses::exp_clamp_count() - c0;
      }
    }
    const double tau_t = c->rep.tau;

    std::vector<Replica> reps(static_cast<size_t>(K), c->rep);
    dist::Fabric fabric(K);
    auto body = [&](int k) {
      Replica& rep = reps[static_cast<size_t>(k)];
      std::vector<int> local_idx(ids + k * Bl, ids + k * Bl + La);
      // trainer.cpp:428-434
      Vector t1_loc(La), t2_loc(La);
      if (indiv) {
        c->itemp.snapshot(local_idx, t1_loc, t2_loc);
      } else {
        t1_loc.setConstant(rep.tau);
        t2_loc.setConstant(rep.tau);
      }
      // trainer.cpp:435-445
      Vector g1_loc, g2_loc;
      engine::g_values(e1g, e2g, t1_loc, t2_loc, k * Bl, La, g1_loc, g2_loc);
      Vector u1_loc(Bl), u2_loc(Bl);
      u1_loc.setConstant(1.0);  // only read for un-sampled anchors in the bounded sample mode
      u2_loc.setConstant(1.0);
      if (track_u) {
        for (int r = 0; r < La; ++r) c->utable->update(local_idx[r], g1_loc[r], g2_loc[r], gamma, k, t);
        Vector a, b;
        c->utable->snapshot(local_idx, t, a, b);
        for (int r = 0; r < La; ++r) { u1_loc[r] = a[r]; u2_loc[r] = b[r]; }
      }
      // trainer.cpp:447-491 (FastCLIP all-gather reduction)
      engine::PairWeights weights;
      Vector u1g(B), u2g(B), tau1g(B), tau2g(B);
      if (v == OC_OPENCLIP_MBCL) {
        Vector tau_all = Vector::Constant(B, rep.tau);
        engine::g_values(e1g, e2g, tau_all, tau_all, 0, B, u1g, u2g);
        weights = engine::weights_mbcl(u1g, u2g, B, rep.tau);
      } else {
        std::vector<double> pay(2u * Bl);
        for (int r = 0; r < Bl; ++r) { pay[r] = u1_loc[r]; pay[Bl + r] = u2_loc[r]; }
        const std::vector<double> g = fabric.all_gather(k, "u-gather", pay);
        for (int w = 0; w < K; ++w)
          for (int r = 0; r < Bl; ++r) {
            u1g[w * Bl + r] = g[w * 2 * Bl + r];
            u2g[w * Bl + r] = g[w * 2 * Bl + Bl + r];
          }
        if (indiv) {
          std::vector<double> tp(2u * Bl, 1.0);
          for (int r = 0; r < La; ++r) { tp[r] = t1_loc[r]; tp[Bl + r] = t2_loc[r]; }
          const std::vector<double> tg = fabric.all_gather(k, "tau-gather", tp);
          for (int w = 0; w < K; ++w)
            for (int r = 0; r < Bl; ++r) {
              tau1g[w * Bl + r] = tg[w * 2 * Bl + r];
              tau2g[w * Bl + r] = tg[w * 2 * Bl + Bl + r];
            }
          weights = engine::weights_individual_tau(u1g, u2g, tau1g, tau2g, eps);
        } else {
          bool scaled = c->cfg.scale_by_tau != 0;
          weights = engine::weights_global_tau(u1g, u2g, rep.tau, eps, scaled);
        }
      }
      // trainer.cpp:521-524
      const engine::Cotangents cot =
          engine::embedding_cotangents(e1g, e2g, weights, k * Bl, La, engine::Parts::both);
      // trainer.cpp:555-589
      double gtl = 0.0;
      if (v == OC_SOGCLR || v == OC_FASTCLIP_V1) {
      } else if (indiv) {
        const auto grads = engine::grad_tau_individual(e1g, e2g, u1g, u2g, tau1g, tau2g, k * Bl, La,
                                                       eps, c->cfg.rho, c->cfg.n_train);
        for (const auto& g : grads) {
          out->gtau1[k * Bl + g.local_row] = g.g_tau1;
          out->gtau2[k * Bl + g.local_row] = g.g_tau2;
          c->itemp.update(local_idx[g.local_row], g.g_tau1, g.g_tau2, c->cfg.tau_lr, c->adam, k,
                          c->utable->owners());
        }
      } else {
        if (v == OC_OPENCLIP_MBCL) gtl = engine::grad_tau_mbcl(e1g, e2g, u1g, u2g, k * Bl, La, rep.tau);
        else if (v == OC_FASTCLIP_V0) gtl = engine::grad_tau_unscaled(e1g, e2g, u1g, u2g, k * Bl, La, rep.tau, eps);
        else gtl = engine::grad_tau_margin(e1g, e2g, u1g, u2g, k * Bl, La, rep.tau, eps, c->cfg.rho);
        const double gtau = fabric.all_reduce_mean_scalar(k, "tau-reduce", gtl);
        double lr = c->cfg.tau_lr;
        if (c->cfg.lr_decay_enabled) lr *= rep.latch.modifier(rep.tau);
        rep.tau = opt::temperature_step(rep.tau_adam, rep.tau, gtau, lr, c->adam, c->cfg.tau0);
        if (k == 0) out->gtau = gtau;
      }
      out->gtau_local[k] = gtl;
      // outputs (rank k's rows)
      for (int r = 0; r < La; ++r) {
        const int i = k * Bl + r;
        out->g1[i] = g1_loc[r];
        out->g2[i] = g2_loc[r];
        out->t1[i] = t1_loc[r];
        out->t2[i] = t2_loc[r];
        for (int q = 0; q < d; ++q) {
          out->dE1[static_cast<size_t>(i) * d + q] = cot.d_e1(r, q);
          out->dE2[static_cast<size_t>(i) * d + q] = cot.d_e2(r, q);
        }
      }
      for (int i = 0; i < B; ++i) {
        if (i / Bl == k) { out->u1[i] = u1g[i]; out->u2[i] = u2g[i]; }
      }
    };
    fabric.run_workers(body);
    c->rep = reps[0];
    out->tau_new = c->rep.tau;
    if (v == OC_SOGCLR || v == OC_FASTCLIP_V1 || indiv) out->gtau = 0.0;

    // Exact batch loss at tau^t (losses.cpp:126-180), as the trainer evaluates per epoch.
    out->loss = 0.0;
    if (want_loss) {
      if (v == OC_OPENCLIP_MBCL) out->loss = losses::eval_mbcl(e1g, e2g, tau_t);
      else if (indiv) out->loss = losses::eval_rgcl(e1g, e2g, from_array(out->t1, B), from_array(out->t2, B), eps, c->cfg.rho);
      else if (v == OC_FASTCLIP_V3) out->loss = losses::eval_rgclg(e1g, e2g, tau_t, eps, c->cfg.rho);
      else out->loss = losses::eval_gcl(e1g, e2g, tau_t, eps);
    }
    return OC_OK;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

int ref_step(void* h, int K, int B, int d, const double* E1, const double* E2, const int32_t* ids,
             double gamma, double eps, oc_step_out* out) {
  return ref_step_ex(h, K, B, d, E1, E2, ids, gamma, eps, out, 0, 1);
}

// ---- per-function entry points (reference functions on row-major inputs) ----
int ref_g_values(int B, int d, const double* E1, const double* E2, const double* t1_local,
                 const double* t2_local, int lo, int cnt, double* g1, double* g2) {
  try {
    Vector a, b;
    engine::g_values(from_rows(E1, B, d), from_rows(E2, B, d), from_array(t1_local, cnt),
                     from_array(t2_local, cnt), lo, cnt, a, b);
    std::memcpy(g1, a.data(), 8u * cnt);
    std::memcpy(g2, b.data(), 8u * cnt);
    return OC_OK;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

int ref_embedding_cotangents(int B, int d, const double* E1, const double* E2, const double* w1,
                             const double* w2, const double* t1, const double* t2, int lo,
                             int cnt, double* dE1, double* dE2) {
  try {
    engine::PairWeights w{from_array(w1, B), from_array(w2, B), from_array(t1, B), from_array(t2, B)};
    const engine::Cotangents cot =
        engine::embedding_cotangents(from_rows(E1, B, d), from_rows(E2, B, d), w, lo, cnt);
    to_rows(cot.d_e1, dE1);
    to_rows(cot.d_e2, dE2);
    return OC_OK;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

double ref_eval_gcl(int B, int d, const double* E1, const double* E2, double tau, double eps) {
  return losses::eval_gcl(from_rows(E1, B, d), from_rows(E2, B, d), tau, eps);
}
double ref_eval_rgcl(int B, int d, const double* E1, const double* E2, const double* t1,
                     const double* t2, double eps, double rho) {
  return losses::eval_rgcl(from_rows(E1, B, d), from_rows(E2, B, d), from_array(t1, B),
                           from_array(t2, B), eps, rho);
}
double ref_eval_mbcl(int B, int d, const double* E1, const double* E2, double tau) {
  return losses::eval_mbcl(from_rows(E1, B, d), from_rows(E2, B, d), tau);
}
double ref_safe_exp(double x) { return losses::safe_exp(x); }
unsigned long long ref_exp_clamp_count(void) { return losses::exp_clamp_count(); }
double ref_gamma_cosine(long long t, long long ipe, long long decay, double gmin) {
  sched::GammaSchedule g;
  g.kind = sched::GammaSchedule::Kind::cosine;
  g.iters_per_epoch = ipe;
  g.decay_epochs = decay;
  g.gamma_min = gmin;
  return g.at(t);
}
int ref_temperature_step(double* m, double* v, int64_t* step, double tau, double grad, double lr,
                         double b1, double b2, double eps, double tau0, double* out) {
  try {
    opt::ScalarAdam st{*m, *v, *step};
    opt::AdamConfig cfg;
    cfg.beta1 = b1; cfg.beta2 = b2; cfg.eps = eps; cfg.weight_decay = 0.123;  // pinned to 0 inside
    *out = opt::temperature_step(st, tau, grad, lr, cfg, tau0);
    *m = st.m; *v = st.v; *step = st.step;
    return OC_OK;
  } catch (...) {
    return status_of(std::current_exception());
  }
}
// Times one reference S product (losses::pairwise_similarity) for the baseline model.
double ref_similarity_checksum(int B, int d, const double* E1, const double* E2) {
  const Matrix s = losses::pairwise_similarity(from_rows(E1, B, d), from_rows(E2, B, d));
  double acc = 0.0;
  for (Eigen::Index i = 0; i < s.rows(); ++i) acc += s(i, i);
  return acc;
}

}  // extern "C"
