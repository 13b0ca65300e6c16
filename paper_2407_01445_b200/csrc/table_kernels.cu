// table_kernels.cu -- the per-anchor (O(B)) kernels of the FastCLIP loss step.
//
// These are latency-bound gather/scatter and scalar kernels (no tensor-core shape):
//   fc_prep_kernel        S_ii = <E1_i, E2_i> and the row-norm bounds for the global batch;
//                         tau^t snapshot (global tau or IndividualTemp by id, state.cpp:112-122)
//                         for the local anchors -> pass-1 row parameters
//   fc_anchor_kernel      per local anchor: u^{t-1} gather by id (before its grid wait), then
//                         the fixed-order reduction of the pass-1 partials -> g
//                         (engine.cpp:151-176), UTable EMA + snapshot (state.cpp:45-71),
//                         PairWeights (engine.cpp:37-75), pass-2 parameters, r_i, the local
//                         tau-gradient / loss terms and the packed payload (+ block partials)
//   fc_weights_kernel     K > 1, after the payload all-gather: pass-2 parameters of every
//                         anchor of G and the u replica update for the other ranks' ids
//   fc_reduce_kernel      fixed-order sum of the (gathered) block partials -> G_tau, loss, and
//                         temperature_step (optimizers.cpp:65-83) with the TauLrLatch
//   fc_indiv_update_kernel  v2: IndividualTemp::update for every id of the global batch
//                         (state.cpp:124-131), replicated identically on every rank
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "table_kernels.cuh"
#include "anchor_device.cuh"

namespace fc {


// Warp per global anchor w: S_ww = <E1_w, E2_w> (fp32 from bf16); the warps of this rank's
// anchors also snapshot tau^t (global tau, or IndividualTemp by id, state.cpp:112-122) and
// emit the pass-1 row parameters.
__global__ void fc_prep_kernel(const __nv_bfloat16* __restrict__ e1, const __nv_bfloat16* __restrict__ e2,
                               StepArgs a, double gamma, double eps, unsigned long long seq) {
  // pass 1 (programmatic launch) may take SMs now: its operand loads and MMAs do not read
  // anything prep writes; its epilogue waits for this grid (griddepcontrol.wait)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (kProfStamps && a.dbg && threadIdx.x == 0) {   // debug timeline: first entry / last exit of the grid
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMin(reinterpret_cast<unsigned long long*>(a.dbg + 8 * 640), static_cast<unsigned long long>(t));
  }
  if (w == 0 && lane == 0) {
    *a.clamps = 0ull;
    *a.step_tag = seq;   // tags this step's duplicate-id set (pass 1 inserts the ids)
    // the step scalars arrive as kernel parameters (updated in the replayed graph per step,
    // no host-to-device copy) and are published for the later kernels of the step
    double* sc = const_cast<double*>(a.scal);
    sc[0] = gamma;
    sc[1] = eps;
  }
  // warp w covers row w of [prep_row0, prep_row0 + prep_rows) (e1 / e2 point at that range)
  const bool valid = w < a.prep_rows;
  const int wl = valid ? w : 0;
  const int wg = a.prep_row0 + w;   // global anchor index
  const int r = wg - a.row0;
  const bool lead = valid && lane == 0 && r >= 0 && r < a.Bl;   // this rank's anchor, lane 0
  const uint4* x4 = reinterpret_cast<const uint4*>(e1 + static_cast<size_t>(wl) * a.d);
  const uint4* y4 = reinterpret_cast<const uint4*>(e2 + static_cast<size_t>(wl) * a.d);
  const int nv = valid ? a.d / 8 : 0;
  // the row loads (two per lane at d = 512) and the id load are all issued before any use
  constexpr int kPre = 2;
  uint4 xs[kPre], ys[kPre];
#pragma unroll
  for (int i = 0; i < kPre; ++i) {
    const int v = lane + 32 * i;
    xs[i] = v < nv ? __ldg(x4 + v) : make_uint4(0u, 0u, 0u, 0u);
    ys[i] = v < nv ? __ldg(y4 + v) : make_uint4(0u, 0u, 0u, 0u);
  }
  int id = lead ? a.ids[r] : 0;
  if (lead && (id < 0 || id >= a.n_train)) {                         // UTable::update range check (state.cpp:46)
    atomicCAS(a.err, 0, kErrShape);             // ShapeError; the table is not touched at this id
    id = 0;
  }
  float acc = 0.f, n1 = 0.f, n2 = 0.f;
  auto accum = [&](const uint4& x, const uint4& y) {
    const uint32_t xx[4] = {x.x, x.y, x.z, x.w};
    const uint32_t yy[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const float2 fx = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xx[t]));
      const float2 fy = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&yy[t]));
      acc = fmaf(fx.x, fy.x, acc);
      acc = fmaf(fx.y, fy.y, acc);
      n1 = fmaf(fx.x, fx.x, fmaf(fx.y, fx.y, n1));
      n2 = fmaf(fy.x, fy.x, fmaf(fy.y, fy.y, n2));
    }
  };
  // u^{t-1} / tau^t of the anchor's id: gathered here, off the table kernel's dependent chain
  // tau^t of the anchor's id (pass 1 needs kappa_i); u^{t-1} is gathered by the per-anchor kernel
  double t1 = 0.0, t2 = 0.0;
  if (lead) {
    if (a.individual) { t1 = a.tau1_tab[id]; t2 = a.tau2_tab[id]; }
    else { t1 = t2 = a.tau_state->tau; }
  }
#pragma unroll
  for (int i = 0; i < kPre; ++i) accum(xs[i], ys[i]);
  for (int v = lane + 32 * kPre; v < nv; v += 32) accum(__ldg(x4 + v), __ldg(y4 + v));   // d > 512
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    acc += __shfl_xor_sync(0xffffffffu, acc, o);
    n1 += __shfl_xor_sync(0xffffffffu, n1, o);
    n2 += __shfl_xor_sync(0xffffffffu, n2, o);
  }
  // norm bounds for the clamp-free fast paths of the similarity kernels (non-negative floats
  // order like their bit patterns): block max first, one atomic per block
  __shared__ float bmax[2][32];
  const int wid = threadIdx.x >> 5;
  if (lane == 0) { bmax[0][wid] = n1; bmax[1][wid] = n2; }
  __syncthreads();
  if (threadIdx.x < 2) {
    float m = 0.f;
    for (int k = 0; k < static_cast<int>(blockDim.x >> 5); ++k) m = fmaxf(m, bmax[threadIdx.x][k]);
    atomicMax(reinterpret_cast<int*>(a.bounds) + threadIdx.x, __float_as_int(m));   // this rank's slot
  }
  if (lane != 0 || !valid) return;
  a.diag[wg] = acc;
  if (!lead) return;
  a.t_loc1[r] = t1;
  a.t_loc2[r] = t2;

  const float k1 = static_cast<float>(kLog2eD / t1), k2 = static_cast<float>(kLog2eD / t2);
  a.rowstat_R[r] = make_float2(k1, -acc * k1);   // y = s * kappa + beta (log2-domain exponent)
  a.rowstat_C[r] = make_float2(k2, -acc * k2);
  if (kProfStamps && a.dbg) {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMax(reinterpret_cast<unsigned long long*>(a.dbg + 8 * 640 + 1), static_cast<unsigned long long>(t));
  }
}

__device__ void block_partials(const StepArgs& a, double ta, double tb, double tl, float kmax);

// Test hook (FC_TEST_DELAY_US): holds this rank's stream for `ns` nanoseconds.
__global__ void fc_delay_kernel(long long ns) {
  long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

// openclip_rs (trainer.cpp:504-518): the anchors of other ranks carry no weights on this rank --
// zero their pass-2 coefficients (the exponent parameters stay, only coef / fac enter Q').
__global__ void fc_rs_mask_kernel(StepArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.B || (i >= a.row0 && i < a.row0 + a.Bl)) return;
  a.coef1[i] = 0.f;
  a.coef2[i] = 0.f;
  a.fac1[i] = 0.f;
  a.fac2[i] = 0.f;
}

// dE += c * reduce-scattered contrast cotangents (engine.cpp:146-149 with the mean's 1/K folded in)
__global__ void fc_axpy2_kernel(float* y1, float* y2, const float* x1, const float* x2, long long n, float c) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    y1[i] = fmaf(c, x1[i], y1[i]);
    y2[i] = fmaf(c, x2[i], y2[i]);
  }
}

// K > 1, after the payload all-gather: thread per anchor of the global batch -> pass-2
// parameters of every anchor (the local ones were written by fc_anchor_kernel as well) and the
// u replica update for the other ranks' ids.
__global__ void fc_weights_kernel(StepArgs a) {
  const double eps = a.scal[1];     // eps_t of this step
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  float kmax = 0.f;
  if (i < a.B) {
    const int k = i / a.Bl;
    const int r = i % a.Bl;
    const double* blk = a.recv + static_cast<size_t>(k) * a.pstride;
    const double u1 = blk[r], u2 = blk[a.Bl + r];
    const double t1 = blk[2 * a.Bl + r], t2 = blk[3 * a.Bl + r];
    const int id = static_cast<int>(blk[4 * a.Bl + r]);
    if (a.track_u && k != a.rank && id >= 0 && id < a.n_train && *a.err != kErrOwnership) {   // keep this rank's u replica equal to the UTable
      a.u1_tab[id] = u1;
      a.u2_tab[id] = u2;
    }
    if (!a.weights_replica_only) {
      const float s_ii = a.diag[i];
      const AnchorParams p = anchor_params(a, u1, u2, t1, t2, a.tau_state->tau, eps);
      store_params(a, i, p, s_ii);
      kmax = fmaxf(p.k1, p.k2);
    }
  }
  if (a.weights_replica_only) return;   // grid-uniform: parameters and kappa max arrived already
  __shared__ float shk[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) kmax = fmaxf(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
  if ((threadIdx.x & 31) == 0) shk[threadIdx.x >> 5] = kmax;
  __syncthreads();
  if (threadIdx.x == 0) {
    float km = 0.f;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) km = fmaxf(km, shk[w]);
    atomicMax(reinterpret_cast<int*>(a.bounds) + 2, __float_as_int(km));   // max kappa (pass-2 fast path)
  }
}

// K = 1: no collective separates the u update from the weights, so a lane group per anchor does
// the partial reduction, and its leader the table update, weights and local terms from
// registers; then the per-block partial sums (reduced off the critical path by fc_reduce_kernel).
__device__ __forceinline__ long long gtime() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(128) fc_anchor_kernel(StepArgs a) {
  long long t_entry = (kProfStamps && a.dbg) ? gtime() : 0;
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) / kGroup;
  const int sub = threadIdx.x % kGroup;
  // the u^{t-1} gather by id (two dependent DRAM round trips) while pass 1 drains
  int id;
  double uo1, uo2;
  anchor_u_old(a, r, id, uo1, uo2);
  asm volatile("griddepcontrol.wait;" ::: "memory");   // pass-1 partials (programmatic launch)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  long long t_wait = (kProfStamps && a.dbg) ? gtime() : 0;
  double ta = 0.0, tb = 0.0, tl = 0.0;
  float kmax = 0.f;
  anchor_work(a, r, sub, id, uo1, uo2, ta, tb, tl, kmax);
  if (kProfStamps && a.dbg && threadIdx.x == 0) a.dbg[blockIdx.x * 8 + 3] = gtime();
  block_partials(a, ta, tb, tl, kmax);
  if (kProfStamps && a.dbg && threadIdx.x == 0) { a.dbg[blockIdx.x * 8 + 0] = t_entry; a.dbg[blockIdx.x * 8 + 1] = t_wait; a.dbg[blockIdx.x * 8 + 4] = gtime(); }
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
  if (learnable_global && *a.err != kErrOwnership) {   // a rejected batch leaves tau as it was
    const double gtau = a.red[0] * (1.0 / static_cast<double>(a.world));
    res->gtau = gtau;
    double lr = a.tau_lr;
    if (a.lr_decay_enabled) {   // TauLrLatch::modifier at the pre-step tau (schedules.hpp:55-58)
      if (tau_t < a.lr_decay_threshold) ts->latched = 1;
      lr *= ts->latched ? a.lr_decay_factor : 1.0;
    }
    if (!isfinite(gtau)) {
      atomicCAS(a.err, 0, kErrNumeric);  // NumericError (optimizers.cpp:67)
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

// Deterministic two-level reduction of the local tau-gradient / loss terms: fixed warp trees
// into per-block partials here (+ the block max of kappa for the pass-2 fast path) ...
__device__ void block_partials(const StepArgs& a, double ta, double tb, double tl, float kmax) {
  __shared__ double sh[3][32];
  __shared__ float shk[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ta += __shfl_xor_sync(0xffffffffu, ta, o);
    tb += __shfl_xor_sync(0xffffffffu, tb, o);
    tl += __shfl_xor_sync(0xffffffffu, tl, o);
    kmax = fmaxf(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
  }
  if (lane == 0) { sh[0][wid] = ta; sh[1][wid] = tb; sh[2][wid] = tl; shk[wid] = kmax; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double b0 = 0.0, b1 = 0.0, b2 = 0.0;
    float km = 0.f;
    for (int w = 0; w < nw; ++w) { b0 += sh[0][w]; b1 += sh[1][w]; b2 += sh[2][w]; km = fmaxf(km, shk[w]); }
    atomicMax(reinterpret_cast<int*>(a.bounds) + 2, __float_as_int(km));   // max kappa, this rank's slot
    double* bp = a.blockpart + 3 * blockIdx.x;
    bp[0] = b0; bp[1] = b1; bp[2] = b2;
  }
}

// ... and the sum of the block partials in a fixed order by ONE WARP (lane t takes blocks
// t, t + 32, ... then a fixed xor tree) in a separate kernel: it forms G_tau,k
// (engine.cpp:208-238) and, when no all-reduce separates them (K = 1), runs the temperature
// step. Nothing on the gradient path waits for it; a single warp without shared memory fits
// beside a persistent similarity CTA, so it never delays the pass-2 launch.
__global__ void __launch_bounds__(32) fc_reduce_kernel(StepArgs a) {
  // rank by rank in rank order (identical arithmetic on every rank, so the replicated tau
  // stays bit-identical): G_tau,k from rank k's block partials (engine.cpp:208-238), summed
  // over k -- the all_reduce_mean_scalar of trainer.cpp:572 without a collective
  double gsum = 0.0, lsum = 0.0;
  for (int k = 0; k < a.world; ++k) {
    const double* bp0 = a.recv + static_cast<size_t>(k) * a.pstride + 7 * static_cast<size_t>(a.Bl);
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int b = threadIdx.x; b < a.nblk; b += 32) {
      const double* bp = bp0 + 3 * b;
      s0 += bp[0]; s1 += bp[1]; s2 += bp[2];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    const double bl = static_cast<double>(a.Bl);
    const double unscaled = s0 / bl;
    double gtl = unscaled;                                                   // v0 / MBCL
    if (a.variant == 6) gtl = s1 / bl + 2.0 * a.rho + a.tau_state->tau * unscaled;  // v3
    gsum += gtl;
    lsum += s2;
  }
  if (threadIdx.x != 0) return;
  a.red[0] = gsum;   // sum over ranks; finalize_step applies the 1/K of the mean (fabric.cpp:73-83)
  a.red[1] = lsum;   // loss numerator over the global batch
  finalize_step(a);
}

// v2 / iSogCLR: IndividualTemp::update for every id of the global batch (state.cpp:124-131);
// each rank applies the same updates in the same arithmetic -> identical table replicas.
__global__ void fc_indiv_update_kernel(StepArgs a) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.B || *a.err == kErrOwnership) return;   // a rejected batch writes no table entry
  const int k = i / a.Bl;
  const int r = i % a.Bl;
  const double* blk = a.recv + static_cast<size_t>(k) * a.pstride;
  const int id = static_cast<int>(blk[4 * a.Bl + r]);
  if (id < 0 || id >= a.n_train) return;   // rejected by its owner's prep (ShapeError)
  const double gts[2] = {blk[5 * a.Bl + r], blk[6 * a.Bl + r]};
  double* taus[2] = {a.tau1_tab, a.tau2_tab};
  double* ms[2] = {a.m1_tab, a.m2_tab};
  double* vs[2] = {a.v1_tab, a.v2_tab};
  long long* ss[2] = {a.s1_tab, a.s2_tab};
  for (int t = 0; t < 2; ++t) {
    const double g = gts[t];
    if (!isfinite(g)) { atomicCAS(a.err, 0, kErrNumeric); return; }
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

namespace fc {

// ---- stateless engine entry points (fc_g_values): engine::g_values + dtau_sums ----

// Warp per global row w of [0, B): norm maxima of E1 / E2 rows into bounds[0..1] (the
// similarity kernel's clamp-free fast-path test); rows of the local slice [lo, lo + cnt) also
// get S_ww and their pass-1 row parameters {kappa = log2(e)/t, beta = -S_ww kappa} at the
// caller's temperatures (engine.cpp:151-176 takes t per local anchor).
__global__ void fc_rows_kernel(const __nv_bfloat16* __restrict__ e1, const __nv_bfloat16* __restrict__ e2, int B,
                               int d, int lo, int cnt, const double* __restrict__ t1, const double* __restrict__ t2,
                               float2* rowstat_R, float2* rowstat_C, float* bounds, float* diag) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  float acc = 0.f, n1 = 0.f, n2 = 0.f;
  if (w < B) {
    const __nv_bfloat162* x = reinterpret_cast<const __nv_bfloat162*>(e1 + static_cast<size_t>(w) * d);
    const __nv_bfloat162* y = reinterpret_cast<const __nv_bfloat162*>(e2 + static_cast<size_t>(w) * d);
    for (int k = lane; k < d / 2; k += 32) {
      const float2 fx = __bfloat1622float2(x[k]), fy = __bfloat1622float2(y[k]);
      acc = fmaf(fx.x, fy.x, fmaf(fx.y, fy.y, acc));
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
  if (lane != 0 || w >= B) return;
  atomicMax(reinterpret_cast<int*>(bounds) + 0, __float_as_int(n1));   // non-negative floats order like ints
  atomicMax(reinterpret_cast<int*>(bounds) + 1, __float_as_int(n2));
  if (diag) diag[w] = acc;
  const int r = w - lo;
  if (r < 0 || r >= cnt) return;
  const float k1 = static_cast<float>(kLog2eD / t1[r]), k2 = static_cast<float>(kLog2eD / t2[r]);
  rowstat_R[r] = make_float2(k1, -acc * k1);
  rowstat_C[r] = make_float2(k2, -acc * k2);
}

// Thread per local row: fixed-order fp64 sum of the row's pass-1 partials of both segments ->
// g = sum e / (B-1) (engine.cpp:176) and dsum = -(sum (s - S_ii) e) / (t^2 (B-1))
// (engine.cpp:198-205; pass 1 accumulates y e with y = (s - S_ii) kappa).
__global__ void fc_gsum_kernel(const float2* __restrict__ pR, const float2* __restrict__ pC, int nparts, int cnt,
                               int B, const float2* __restrict__ rsR, const float2* __restrict__ rsC,
                               const double* __restrict__ t1, const double* __restrict__ t2, double* g1, double* g2,
                               double* ds1, double* ds2) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= cnt) return;
  double s1 = 0.0, x1 = 0.0, s2 = 0.0, x2 = 0.0;
  for (int q = 0; q < nparts; ++q) {
    const float2 a = pR[static_cast<size_t>(r) * nparts + q], b = pC[static_cast<size_t>(r) * nparts + q];
    s1 += a.x; x1 += a.y; s2 += b.x; x2 += b.y;
  }
  const double inv = 1.0 / static_cast<double>(B - 1);
  g1[r] = s1 * inv;
  g2[r] = s2 * inv;
  if (ds1) {
    const double d1 = x1 / static_cast<double>(rsR[r].x), d2 = x2 / static_cast<double>(rsC[r].x);
    ds1[r] = (-(d1 / (t1[r] * t1[r]))) * inv;
    ds2[r] = (-(d2 / (t2[r] * t2[r]))) * inv;
  }
}

// engine::embedding_cotangents parameters (fc_embedding_cotangents): the pass-2 exponent /
// weight parameters of every anchor a of G from the caller's PairWeights (engine.hpp:29-32):
// kappa = log2(e)/t_a, beta = -S_aa kappa, coef = w_a / t_a, fac = coef 2^beta; the kappa
// maximum goes to bounds[2]. Arrays are zero-padded to whole 256-column tiles by the caller.
__global__ void fc_pair_params_kernel(const float* __restrict__ diag, const double* __restrict__ w1,
                                      const double* __restrict__ w2, const double* __restrict__ t1,
                                      const double* __restrict__ t2, int B, float* kap1, float* bet1, float* coef1,
                                      float* fac1, float* kap2, float* bet2, float* coef2, float* fac2,
                                      float* bounds) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B) return;
  AnchorParams p;
  p.t1 = t1[i];
  p.t2 = t2[i];
  p.c1 = w1[i] / p.t1;
  p.c2 = w2[i] / p.t2;
  p.k1 = static_cast<float>(kLog2eD / p.t1);
  p.k2 = static_cast<float>(kLog2eD / p.t2);
  const float s_ii = diag[i];
  const float b1 = -s_ii * p.k1, b2 = -s_ii * p.k2;
  const float c1 = static_cast<float>(p.c1), c2 = static_cast<float>(p.c2);
  kap1[i] = p.k1; bet1[i] = b1; coef1[i] = c1; fac1[i] = c1 * exp2f(b1);
  kap2[i] = p.k2; bet2[i] = b2; coef2[i] = c2; fac2[i] = c2 * exp2f(b2);
  atomicMax(reinterpret_cast<int*>(bounds) + 2, __float_as_int(fmaxf(p.k1, p.k2)));
}

// r_i = (w1_i/t1_i) S1_i + (w2_i/t2_i) S2_i of the local rows (fixed-order sum of the pass-1
// partials), the anchor-part coefficient of engine.cpp:93-106.
__global__ void fc_rcoef_kernel(const float2* __restrict__ pR, const float2* __restrict__ pC, int nparts, int cnt,
                                int lo, const double* __restrict__ w1, const double* __restrict__ w2,
                                const double* __restrict__ t1, const double* __restrict__ t2, float* rcoef) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= cnt) return;
  double s1 = 0.0, s2 = 0.0;
  for (int q = 0; q < nparts; ++q) {
    s1 += pR[static_cast<size_t>(r) * nparts + q].x;
    s2 += pC[static_cast<size_t>(r) * nparts + q].x;
  }
  const int i = lo + r;
  rcoef[r] = static_cast<float>(w1[i] / t1[i] * s1 + w2[i] / t2[i] * s2);
}

}  // namespace fc
