// anchor_device.cuh -- the per-anchor arithmetic of the FastCLIP step as device functions,
// shared by fc_anchor_kernel (table_kernels.cu) and the pass-2 kernel's fused anchor prologue
// (sim_kernel.cu). Pure functions of register values; the loads happen up front and the
// stores at the end, so one anchor is a single memory round trip.
#pragma once

#include <cstdint>

#include "table_kernels.cuh"

namespace fc {

namespace anchor_detail {
constexpr double kLog2eD = 1.4426950408889634073599;
}
using anchor_detail::kLog2eD;

// Anchors per warp of the per-anchor kernels: kGroup lanes reduce one anchor's partials, and
// the scalar fp64 chain then runs on the group leaders, four anchors per warp instruction.
constexpr int kGroup = kAnchorLanes;

// Fixed-order (group-lane-strided + xor tree) reduction of one anchor's pass-1 partials; every
// lane of the warp must call it (valid = false contributes nothing).
// The anchor's row partials (n_r, contiguous) and column partials (n_c, stride cs) are summed
// by the kGroup lanes in a fixed order (lane `sub` takes q = sub, sub + kGroup, ... of each
// list, row list first). The loads of both lists go out 16 at a time from one virtual index
// space, so a lane waits for ~2 memory round trips instead of one per 8 loads.
__device__ __forceinline__ void sum_two(const float2* __restrict__ rp, int n_r, const float2* __restrict__ cp,
                                        size_t cs, int n_c, int sub, double& s1, double& x1, double& s2,
                                        double& x2) {
  const int m_r = n_r > sub ? (n_r - sub + kGroup - 1) / kGroup : 0;   // this lane's row items
  const int m_c = n_c > sub ? (n_c - sub + kGroup - 1) / kGroup : 0;
  const int m = m_r + m_c;
  for (int t0 = 0; t0 < m; t0 += 16) {
    float2 v[16];
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int i = t0 + t;
      v[t] = i < m_r ? __ldg(rp + sub + i * kGroup)
           : (i < m ? __ldg(cp + (sub + (i - m_r) * kGroup) * cs) : make_float2(0.f, 0.f));
    }
#pragma unroll
    for (int t = 0; t < 16; ++t) {
      const int i = t0 + t;
      if (i < m_r) { s1 += v[t].x; x1 += v[t].y; }
      else if (i < m) { s2 += v[t].x; x2 += v[t].y; }
    }
  }
}

__device__ __forceinline__ void reduce_partials(const StepArgs& a, int r, bool valid, int sub, double& s1,
                                                double& x1, double& s2, double& x2) {
  const int nparts = a.n_jt * 4;
  s1 = 0.0; x1 = 0.0; s2 = 0.0; x2 = 0.0;
  if (valid) {
    const float2* rp = a.partial_R + static_cast<size_t>(r) * nparts;
    if (a.col_slots > 0) {   // fused pass 1: column statistics of S, [B/32][slots][32]
      const int j = a.row0 + r;
      sum_two(rp, nparts, a.col_partial + static_cast<size_t>(j >> 5) * a.col_slots * 32 + (j & 31), 32,
              a.col_slots, sub, s1, x1, s2, x2);
    } else {
      sum_two(rp, nparts, a.partial_C + static_cast<size_t>(r) * nparts, 1, nparts, sub, s1, x1, s2, x2);
    }
  }
#pragma unroll
  for (int o = kGroup / 2; o > 0; o >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    x1 += __shfl_xor_sync(0xffffffffu, x1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    x2 += __shfl_xor_sync(0xffffffffu, x2, o);
  }
}

struct TableVals {
  double dx1, dx2, g1, g2, u1, u2;
};

// g (engine.cpp:151-176) and the fp64 EMA of the u entry (state.cpp:52-53); pass 1
// accumulates sum(y e) with y = (s - S_ii) kappa, so dx divides kappa back out.
__device__ __forceinline__ TableVals table_math(const StepArgs& a, double s1, double x1, double s2, double x2,
                                                float kap_r, float kap_c, double uo1, double uo2, double gamma) {
  TableVals v;
  v.dx1 = x1 / static_cast<double>(kap_r);
  v.dx2 = x2 / static_cast<double>(kap_c);
  const double inv = 1.0 / static_cast<double>(a.B - 1);
  v.g1 = s1 * inv;   // engine.cpp:176
  v.g2 = s2 * inv;
  v.u1 = v.g1;       // MBCL: the "u" gathered is the current-batch g (trainer.cpp:456)
  v.u2 = v.g2;
  if (a.track_u) {
    v.u1 = (1.0 - gamma) * uo1 + gamma * v.g1;
    v.u2 = (1.0 - gamma) * uo2 + gamma * v.g2;
  }
  return v;
}

struct AnchorParams {
  double c1, c2, t1, t2;
  float k1, k2;
};

// PairWeights of one anchor (engine.cpp:37-75) -> pass-2 exponent / coefficient parameters.
__device__ __forceinline__ AnchorParams anchor_params(const StepArgs& a, double u1, double u2, double t1, double t2,
                                                      double tau, double eps) {
  double w1, w2;
  if (a.variant == 0) {  // MBCL: weights_mbcl (engine.cpp:65-75)
    const double c = 1.0 / static_cast<double>(a.B - 1);
    w1 = 1.0 / (c + u1);
    w2 = 1.0 / (c + u2);
    t1 = t2 = tau;
  } else if (a.individual) {  // weights_individual_tau (engine.cpp:52-63)
    w1 = (1.0 / (eps + u1)) * t1;
    w2 = (1.0 / (eps + u2)) * t2;
  } else {  // weights_global_tau (engine.cpp:37-50)
    w1 = 1.0 / (eps + u1);
    w2 = 1.0 / (eps + u2);
    if (a.scale_by_tau) { w1 *= tau; w2 *= tau; }
    t1 = t2 = tau;
  }
  AnchorParams p;
  p.t1 = t1;
  p.t2 = t2;
  p.c1 = w1 / t1;   // P1 coefficient: w1_a / t1_a  (engine.cpp:104,118)
  p.c2 = w2 / t2;   // P2 coefficient: w2_a / t2_a
  p.k1 = static_cast<float>(kLog2eD / t1);
  p.k2 = static_cast<float>(kLog2eD / t2);
  return p;
}

__device__ __forceinline__ void store_params(const StepArgs& a, int i, const AnchorParams& p, float s_ii) {
  const float b1 = -s_ii * p.k1, b2 = -s_ii * p.k2;
  const float c1 = static_cast<float>(p.c1), c2 = static_cast<float>(p.c2);
  a.kap1[i] = p.k1; a.bet1[i] = b1; a.coef1[i] = c1; a.fac1[i] = c1 * exp2f(b1);
  a.kap2[i] = p.k2; a.bet2[i] = b2; a.coef2[i] = c2; a.fac2[i] = c2 * exp2f(b2);
}

// The four logarithms of an anchor's tau-gradient / loss terms, one per lane of its group:
// lane k of the group evaluates log(arg_k) with arg = {eps + u1, eps + u2, e + g1, e + g2}
// (e = 1/(B-1) for MBCL, eps otherwise).
__device__ __forceinline__ double log_arg(const StepArgs& a, int k, double u1, double u2, double g1, double g2,
                                          double eps) {
  const double e = a.variant == 0 ? 1.0 / static_cast<double>(a.B - 1) : eps;
  return k == 0 ? eps + u1 : k == 1 ? eps + u2 : k == 2 ? e + g1 : e + g2;
}

// Local anchor: tau-gradient and loss terms (engine.cpp:198-266, losses.cpp:126-180) from the
// precomputed logs lu = log(eps + u), lg = log(e + g); v2 writes its per-anchor tau gradients.
__device__ __forceinline__ void local_terms(const StepArgs& a, int r, const AnchorParams& p, double u1, double u2,
                                            double g1, double g2, double dx1, double dx2, double eps, double lu1,
                                            double lu2, double lg1, double lg2, double& ta, double& tb, double& tl) {
  const double t1 = p.t1, t2 = p.t2;
  const double inv = 1.0 / static_cast<double>(a.B - 1);
  const double ds1 = (-(dx1 / (t1 * t1))) * inv;   // engine.cpp:198-205
  const double ds2 = (-(dx2 / (t2 * t2))) * inv;
  if (a.variant == 0) {
    const double c = inv;
    ta = ds1 / (c + g1) + ds2 / (c + g2);                 // grad_tau_mbcl (engine.cpp:261-266)
    tl = lg1 + lg2;                                       // eval_mbcl (losses.cpp:168-180)
  } else if (a.individual) {
    const double inv_n = 1.0 / static_cast<double>(a.n_train);   // engine.cpp:240-259
    a.gt1[r] = inv_n * (lu1 + a.rho + t1 * ds1 / (eps + u1));
    a.gt2[r] = inv_n * (lu2 + a.rho + t2 * ds2 / (eps + u2));
    tl = t1 * (lg1 + a.rho) + t2 * (lg2 + a.rho);          // eval_rgcl
  } else {
    ta = ds1 / (eps + u1) + ds2 / (eps + u2);             // grad_tau_unscaled (engine.cpp:208-224)
    tb = lu1 + lu2;                                       // grad_tau_margin logs (engine.cpp:226-238)
    tl = lg1 + lg2;                                       // eval_gcl (losses.cpp:126-138)
  }
}

__device__ __forceinline__ void store_payload(const StepArgs& a, int r, int id, const TableVals& v, double t1,
                                              double t2) {
  // state.cpp:52-53 EMA, then the snapshot (state.cpp:57-71); a batch with a repeated id (prep
  // flagged FC_ERR_OWNERSHIP) writes no entry
  if (a.track_u && id >= 0 && id < a.n_train && *a.err != kErrOwnership) {
    a.u1_tab[id] = v.u1;
    a.u2_tab[id] = v.u2;
  }
  a.g1[r] = v.g1; a.g2[r] = v.g2;
  a.u1[r] = v.u1; a.u2[r] = v.u2;
  // packed payload [u1 | u2 | t1 | t2 | id] (trainer.cpp:459-487 "u-gather" + "tau-gather")
  double* snd = a.send;
  snd[r] = v.u1;
  snd[a.Bl + r] = v.u2;
  snd[2 * a.Bl + r] = t1;
  snd[3 * a.Bl + r] = t2;
  snd[4 * a.Bl + r] = static_cast<double>(id);
}

// One anchor of this rank (local index r, lane `sub` of its kGroup-lane group): the fixed-order
// partial reduction, g and the u EMA (engine.cpp:151-176, state.cpp:45-71), PairWeights and the
// pass-2 parameters (engine.cpp:37-75), r_i, the local tau-gradient / loss terms (returned for
// the caller's block reduction) and the packed payload. Every lane of the warp must call it.
// u^{t-1} of anchor r's id (uo1 / uo2): loaded by the caller before its grid-dependency wait --
// the tables were last written by the previous step, the ids are the step's input.
__device__ __forceinline__ void anchor_u_old(const StepArgs& a, int r, int& id, double& uo1, double& uo2) {
  const int rr = r < a.Bl ? r : 0;
  id = a.ids[rr];
  const bool ok = id >= 0 && id < a.n_train;   // out of range: prep reports ShapeError, no table access
  uo1 = (a.track_u && ok) ? a.u1_tab[id] : 0.0;
  uo2 = (a.track_u && ok) ? a.u2_tab[id] : 0.0;
}

__device__ __forceinline__ void anchor_work(const StepArgs& a, int r, int sub, int id, double uo1, double uo2,
                                            double& ta, double& tb, double& tl, float& kmax) {
  const bool valid = r < a.Bl;
  const int rr = valid ? r : 0;
  // every load of the anchor first (independent, overlapping the partial loads)
  const double gamma = a.scal[0], eps = a.scal[1];
  const double tau = a.tau_state->tau;
  const float kr = a.rowstat_R[rr].x, kc = a.rowstat_C[rr].x;
  const double t1 = a.t_loc1[rr], t2 = a.t_loc2[rr];
  const float s_ii = a.diag[a.row0 + rr];
  double s1, x1, s2, x2;
  reduce_partials(a, rr, valid, sub, s1, x1, s2, x2);
  if (kProfStamps && a.dbg && threadIdx.x == 0) {   // debug timeline: partials reduced
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    a.dbg[blockIdx.x * 8 + 2] = t;
  }
  // every lane of the group holds the sums: g, u and the weights are evaluated redundantly, and
  // the four logarithms of the anchor's terms run on four lanes at once
  const TableVals v = table_math(a, s1, x1, s2, x2, kr, kc, uo1, uo2, gamma);
  const double lg = log(log_arg(a, sub & 3, v.u1, v.u2, v.g1, v.g2, eps));
  const int base = (threadIdx.x & 31) & ~(kGroup - 1);
  const double lu1 = __shfl_sync(0xffffffffu, lg, base + 0), lu2 = __shfl_sync(0xffffffffu, lg, base + 1);
  const double lg1 = __shfl_sync(0xffffffffu, lg, base + 2), lg2 = __shfl_sync(0xffffffffu, lg, base + 3);
  if (sub == 0 && valid) {
    const AnchorParams p = anchor_params(a, v.u1, v.u2, t1, t2, tau, eps);
    kmax = fmaxf(kmax, fmaxf(p.k1, p.k2));
    local_terms(a, r, p, v.u1, v.u2, v.g1, v.g2, v.dx1, v.dx2, eps, lu1, lu2, lg1, lg2, ta, tb, tl);
    a.rcoef[r] = static_cast<float>(p.c1 * s1 + p.c2 * s2);
    store_params(a, a.row0 + r, p, s_ii);
    a.sum1[r] = s1; a.dx1[r] = v.dx1; a.sum2[r] = s2; a.dx2[r] = v.dx2;
    store_payload(a, r, id, v, t1, t2);
  }
}

}  // namespace fc
