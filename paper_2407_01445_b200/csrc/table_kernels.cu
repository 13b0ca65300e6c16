// table_kernels.cu -- the per-anchor (O(B)) kernels of the FastCLIP loss step.
//
// These are HBM/latency-bound gather/scatter and scalar kernels (no tensor-core shape):
//   fc_diag_kernel        S_ii = <E1_i, E2_i> for the global batch (fp32 from bf16)
//   fc_rowpar_kernel      tau^t snapshot per local anchor (global tau or IndividualTemp
//                         gather by id, state.cpp:112-122) -> pass-1 row parameters
//   fc_table_kernel       fixed-order reduction of the pass-1 partials -> g (engine.cpp:151-176),
//                         UTable EMA + snapshot (state.cpp:45-71), packed all-gather payload
//   fc_weights_kernel     PairWeights for the whole batch (engine.cpp:37-75), pass-2 row/col
//                         parameters, r_i, per-anchor tau-gradient and loss terms
//   fc_reduce_kernel      fixed-order block reduction of the local terms (G_tau, loss)
//   fc_finalize_kernel    all-reduced G_tau -> temperature_step (optimizers.cpp:65-83) with the
//                         TauLrLatch (schedules.hpp:55-58); step scalars
//   fc_indiv_update_kernel  v2: IndividualTemp::update for every id of the global batch
//                         (state.cpp:124-131), replicated identically on every rank
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "table_kernels.cuh"

namespace fc {

namespace {
constexpr double kLog2eD = 1.4426950408889634073599;
}

// Warp per global anchor w: S_ww = <E1_w, E2_w> (fp32 from bf16); the warps of this rank's
// anchors also snapshot tau^t (global tau, or IndividualTemp by id, state.cpp:112-122) and
// emit the pass-1 row parameters.
__global__ void fc_prep_kernel(const __nv_bfloat16* __restrict__ e1, const __nv_bfloat16* __restrict__ e2,
                               StepArgs a) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (w == 0 && lane == 0) *a.clamps = 0ull;
  if (w >= a.B) return;
  const uint4* x4 = reinterpret_cast<const uint4*>(e1 + static_cast<size_t>(w) * a.d);
  const uint4* y4 = reinterpret_cast<const uint4*>(e2 + static_cast<size_t>(w) * a.d);
  float acc = 0.f, n1 = 0.f, n2 = 0.f;
  for (int v = lane; v < a.d / 8; v += 32) {
    const uint4 x = __ldg(x4 + v);
    const uint4 y = __ldg(y4 + v);
    const uint32_t xs[4] = {x.x, x.y, x.z, x.w};
    const uint32_t ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const float2 fx = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xs[t]));
      const float2 fy = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ys[t]));
      acc = fmaf(fx.x, fy.x, acc);
      acc = fmaf(fx.y, fy.y, acc);
      n1 = fmaf(fx.x, fx.x, fmaf(fx.y, fx.y, n1));
      n2 = fmaf(fy.x, fy.x, fmaf(fy.y, fy.y, n2));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    acc += __shfl_xor_sync(0xffffffffu, acc, o);
    n1 += __shfl_xor_sync(0xffffffffu, n1, o);
    n2 += __shfl_xor_sync(0xffffffffu, n2, o);
  }
  if (lane != 0) return;
  // norm bounds for the clamp-free fast paths of the similarity kernels (non-negative floats
  // order like their bit patterns)
  atomicMax(reinterpret_cast<int*>(a.bounds) + 0, __float_as_int(n1));
  atomicMax(reinterpret_cast<int*>(a.bounds) + 1, __float_as_int(n2));
  a.diag[w] = acc;
  const int r = w - a.row0;
  if (r < 0 || r >= a.Bl) return;
  double t1, t2;
  if (a.individual) {
    const int id = a.ids[r];
    t1 = a.tau1_tab[id];
    t2 = a.tau2_tab[id];
  } else {
    t1 = t2 = a.tau_state->tau;
  }
  a.t_loc1[r] = t1;
  a.t_loc2[r] = t2;
  const float k1 = static_cast<float>(kLog2eD / t1), k2 = static_cast<float>(kLog2eD / t2);
  a.rowstat_R[r] = make_float2(k1, -acc * k1);   // y = s * kappa + beta (log2-domain exponent)
  a.rowstat_C[r] = make_float2(k2, -acc * k2);
}

// Warp per local anchor: fixed-order (lane-strided + xor tree) reduction of the pass-1
// partials, then g (engine.cpp:151-176), the fp64 EMA of the owned u entries (state.cpp:52-53)
// and the snapshot (state.cpp:57-71), written straight into the all-gather payload.
__global__ void fc_table_kernel(StepArgs a) {
  const double gamma = a.scal[0];   // gamma_t of this step (device, so the step can be graph-replayed)
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (r >= a.Bl) return;
  const int nparts = a.n_jt * 4;
  const float2* pr = a.partial_R + static_cast<size_t>(r) * nparts;
  const float2* pc = a.partial_C + static_cast<size_t>(r) * nparts;
  double s1 = 0.0, x1 = 0.0, s2 = 0.0, x2 = 0.0;
  for (int q = lane; q < nparts; q += 32) {
    const float2 u = pr[q];
    const float2 v = pc[q];
    s1 += u.x; x1 += u.y;
    s2 += v.x; x2 += v.y;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    x1 += __shfl_xor_sync(0xffffffffu, x1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    x2 += __shfl_xor_sync(0xffffffffu, x2, o);
  }
  if (lane != 0) return;
  // pass 1 accumulates sum(y e) with y = (s - S_ii) kappa: divide back by kappa
  a.sum1[r] = s1; a.dx1[r] = x1 / static_cast<double>(a.rowstat_R[r].x);
  a.sum2[r] = s2; a.dx2[r] = x2 / static_cast<double>(a.rowstat_C[r].x);
  const double inv = 1.0 / static_cast<double>(a.B - 1);
  const double g1 = s1 * inv;   // engine.cpp:176
  const double g2 = s2 * inv;
  a.g1[r] = g1;
  a.g2[r] = g2;
  double u1 = g1, u2 = g2;      // MBCL: the "u" gathered is the current-batch g (trainer.cpp:456)
  const int id = a.ids[r];
  if (a.track_u) {              // state.cpp:52-53 (fp64 EMA), then snapshot (state.cpp:57-71)
    u1 = (1.0 - gamma) * a.u1_tab[id] + gamma * g1;
    u2 = (1.0 - gamma) * a.u2_tab[id] + gamma * g2;
    a.u1_tab[id] = u1;
    a.u2_tab[id] = u2;
  }
  a.u1[r] = u1;
  a.u2[r] = u2;
  // packed payload [u1 | u2 | t1 | t2 | id] (trainer.cpp:459-487 "u-gather" + "tau-gather")
  double* snd = a.send;
  snd[r] = u1;
  snd[a.Bl + r] = u2;
  snd[2 * a.Bl + r] = a.t_loc1[r];
  snd[3 * a.Bl + r] = a.t_loc2[r];
  snd[4 * a.Bl + r] = static_cast<double>(id);
}

__device__ void block_reduce_and_finish(const StepArgs& a, double ta, double tb, double tl);
__device__ __forceinline__ void weights_one(const StepArgs& a, int i, double eps, double& ta, double& tb,
                                            double& tl);

__global__ void fc_weights_kernel(StepArgs a) {
  const double eps = a.scal[1];     // eps_t of this step
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  double ta = 0.0, tb = 0.0, tl = 0.0;
  // every thread reaches the block reduction from the same place (warp-synchronous shuffles)
  if (i < a.B) weights_one(a, i, eps, ta, tb, tl);
  block_reduce_and_finish(a, ta, tb, tl);
}

__device__ __forceinline__ void weights_one(const StepArgs& a, int i, double eps, double& ta, double& tb,
                                            double& tl) {
  const int k = i / a.Bl;
  const int r = i % a.Bl;
  const double* blk = a.recv + static_cast<size_t>(k) * 5 * a.Bl;
  const double u1 = blk[r], u2 = blk[a.Bl + r];
  double t1 = blk[2 * a.Bl + r], t2 = blk[3 * a.Bl + r];
  const double tau = a.tau_state->tau;
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
  const double c1 = w1 / t1;   // P1 coefficient: w1_a / t1_a  (engine.cpp:104,118)
  const double c2 = w2 / t2;   // P2 coefficient: w2_a / t2_a
  const float s_ii = a.diag[i];
  const float k1 = static_cast<float>(kLog2eD / t1);
  const float k2 = static_cast<float>(kLog2eD / t2);
  a.kap1[i] = k1; a.bet1[i] = -s_ii * k1; a.coef1[i] = static_cast<float>(c1);
  a.kap2[i] = k2; a.bet2[i] = -s_ii * k2; a.coef2[i] = static_cast<float>(c2);
  atomicMax(reinterpret_cast<int*>(a.bounds) + 2, __float_as_int(fmaxf(k1, k2)));

  if (k == a.rank) {
    // ---- local anchor: r_i, tau-gradient terms, loss term ----
    a.rcoef[r] = static_cast<float>(c1 * a.sum1[r] + c2 * a.sum2[r]);
    const double inv = 1.0 / static_cast<double>(a.B - 1);
    const double ds1 = (-(a.dx1[r] / (t1 * t1))) * inv;   // engine.cpp:198-205
    const double ds2 = (-(a.dx2[r] / (t2 * t2))) * inv;
    const double g1 = a.g1[r], g2 = a.g2[r];
    if (a.variant == 0) {
      const double c = inv;
      ta = ds1 / (c + g1) + ds2 / (c + g2);                 // grad_tau_mbcl (engine.cpp:261-266)
      tl = log(c + g1) + log(c + g2);                       // eval_mbcl (losses.cpp:168-180)
    } else if (a.individual) {
      const double inv_n = 1.0 / static_cast<double>(a.n_train);   // engine.cpp:240-259
      a.gt1[r] = inv_n * (log(eps + u1) + a.rho + t1 * ds1 / (eps + u1));
      a.gt2[r] = inv_n * (log(eps + u2) + a.rho + t2 * ds2 / (eps + u2));
      tl = t1 * (log(eps + g1) + a.rho) + t2 * (log(eps + g2) + a.rho);  // eval_rgcl
    } else {
      ta = ds1 / (eps + u1) + ds2 / (eps + u2);             // grad_tau_unscaled (engine.cpp:208-224)
      tb = log(eps + u1) + log(eps + u2);                   // grad_tau_margin logs (engine.cpp:226-238)
      tl = log(eps + g1) + log(eps + g2);                   // eval_gcl (losses.cpp:126-138)
    }
  }
}


// trainer.cpp:557-577 for the global-temperature schemes + step scalars for every variant.
__device__ void finalize_step(const StepArgs& a) {
  TauState* ts = a.tau_state;
  const double tau_t = ts->tau;
  const double nB = static_cast<double>(a.B);
  StepResult* res = a.result;
  // exact batch loss at tau^t (losses.cpp:126-180)
  double loss;
  if (a.variant == 0 || a.individual) loss = a.red[1] / nB;
  else loss = tau_t * a.red[1] / nB;
  if (a.variant == 6) loss += 2.0 * a.rho * tau_t;
  res->loss = loss;
  res->gtau = 0.0;
  res->clamps = *a.clamps;
  const bool learnable_global = (a.variant == 0 || a.variant == 3 || a.variant == 6);
  if (learnable_global) {
    const double gtau = a.red[0] * (1.0 / static_cast<double>(a.world));
    res->gtau = gtau;
    double lr = a.tau_lr;
    if (a.lr_decay_enabled) {   // TauLrLatch::modifier at the pre-step tau (schedules.hpp:55-58)
      if (tau_t < a.lr_decay_threshold) ts->latched = 1;
      lr *= ts->latched ? a.lr_decay_factor : 1.0;
    }
    if (!isfinite(gtau)) {
      *a.err = 9;  // NumericError (optimizers.cpp:67)
    } else {       // scalar_adamw_step with weight decay 0, then projection (optimizers.cpp:65-83)
      ts->m = a.beta1 * ts->m + (1.0 - a.beta1) * gtau;
      ts->v = a.beta2 * ts->v + (1.0 - a.beta2) * gtau * gtau;
      const double c1 = 1.0 - pow(a.beta1, static_cast<double>(ts->step + 1));
      const double c2 = 1.0 - pow(a.beta2, static_cast<double>(ts->step + 1));
      ts->step += 1;
      const double rr = (ts->m / c1) / (sqrt(ts->v / c2) + a.adam_eps);
      const double next = tau_t - lr * (rr + 0.0 * tau_t);
      ts->tau = next < a.tau0 ? a.tau0 : next;
    }
  }
  res->tau = ts->tau;
  res->latched = ts->latched;
  res->err = *a.err;
}

// Deterministic two-level reduction of the local tau-gradient / loss terms: fixed warp
// trees into per-block partials, then the LAST block to finish (threadfence + ticket) sums
// the partials in block order, forms G_tau,k (engine.cpp:208-238) and, when no all-reduce
// separates them (K = 1), runs the temperature step.
__device__ void block_reduce_and_finish(const StepArgs& a, double ta, double tb, double tl) {
  __shared__ double sh[3][32];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ta += __shfl_xor_sync(0xffffffffu, ta, o);
    tb += __shfl_xor_sync(0xffffffffu, tb, o);
    tl += __shfl_xor_sync(0xffffffffu, tl, o);
  }
  if (lane == 0) { sh[0][wid] = ta; sh[1][wid] = tb; sh[2][wid] = tl; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double b0 = 0.0, b1 = 0.0, b2 = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) { b0 += sh[0][w]; b1 += sh[1][w]; b2 += sh[2][w]; }
    double* bp = a.blockpart + 3 * blockIdx.x;
    bp[0] = b0; bp[1] = b1; bp[2] = b2;
    __threadfence();
    const unsigned ticket = atomicAdd(a.counter, 1u);
    last = ticket == gridDim.x - 1;
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  __threadfence();
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (unsigned b = 0; b < gridDim.x; ++b) {
    const volatile double* bp = a.blockpart + 3 * b;
    s0 += bp[0]; s1 += bp[1]; s2 += bp[2];
  }
  *a.counter = 0u;   // re-arm for the next step
  const double bl = static_cast<double>(a.Bl);
  const double unscaled = s0 / bl;
  double gtl = unscaled;                                                   // v0 / MBCL
  if (a.variant == 6) gtl = s1 / bl + 2.0 * a.rho + a.tau_state->tau * unscaled;  // v3
  a.red[0] = gtl;   // all-reduced (sum) across ranks, then * 1/K (fabric.cpp:73-83)
  a.red[1] = s2;    // loss numerator, summed across ranks
  if (a.fuse_finalize) finalize_step(a);
}

__global__ void fc_finalize_kernel(StepArgs a) {
  if (threadIdx.x == 0 && blockIdx.x == 0) finalize_step(a);
}

// v2 / iSogCLR: IndividualTemp::update for every id of the global batch (state.cpp:124-131);
// each rank applies the same updates in the same arithmetic -> identical table replicas.
__global__ void fc_indiv_update_kernel(StepArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.B) return;
  const int k = i / a.Bl;
  const int r = i % a.Bl;
  const int id = static_cast<int>(a.recv[static_cast<size_t>(k) * 5 * a.Bl + 4 * a.Bl + r]);
  const double gts[2] = {a.gt_recv[static_cast<size_t>(k) * 2 * a.Bl + r],
                         a.gt_recv[static_cast<size_t>(k) * 2 * a.Bl + a.Bl + r]};
  double* taus[2] = {a.tau1_tab, a.tau2_tab};
  double* ms[2] = {a.m1_tab, a.m2_tab};
  double* vs[2] = {a.v1_tab, a.v2_tab};
  long long* ss[2] = {a.s1_tab, a.s2_tab};
  for (int t = 0; t < 2; ++t) {
    const double g = gts[t];
    if (!isfinite(g)) { *a.err = 9; return; }
    double m = ms[t][id], v = vs[t][id];
    const long long st = ss[t][id];
    m = a.beta1 * m + (1.0 - a.beta1) * g;
    v = a.beta2 * v + (1.0 - a.beta2) * g * g;
    const double c1 = 1.0 - pow(a.beta1, static_cast<double>(st + 1));
    const double c2 = 1.0 - pow(a.beta2, static_cast<double>(st + 1));
    const double rr = (m / c1) / (sqrt(v / c2) + a.adam_eps);
    const double tau = taus[t][id];
    const double next = tau - a.tau_lr * (rr + 0.0 * tau);
    ms[t][id] = m;
    vs[t][id] = v;
    ss[t][id] = st + 1;
    taus[t][id] = next < a.tau0 ? a.tau0 : next;
  }
}

}  // namespace fc
