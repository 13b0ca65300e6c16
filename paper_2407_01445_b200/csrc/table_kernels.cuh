// table_kernels.cuh -- device state and argument block of the per-anchor kernels.
#pragma once

#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace fc {

// Replica scalar state of the global temperature (trainer.cpp:245-254), device resident.
struct TauState {
  double tau;
  double m, v;
  long long step;
  int latched;
  int pad;
};

// Scalars of one step, copied to pinned host memory at the end of the step.
struct StepResult {
  double loss;
  double gtau;
  double tau;
  unsigned long long clamps;
  int latched;
  int err;
};

// lanes per anchor in fc_anchor_kernel (partial reduction width; the leader runs the fp64 chain)
constexpr int kAnchorLanes = 16;

struct StepArgs {
  // shapes / config
  int B, Bl, d, world, rank, row0, n_jt;
  int variant, individual, track_u, scale_by_tau, lr_decay_enabled;
  long long n_train;
  double rho, tau_lr, tau0, beta1, beta2, adam_eps, lr_decay_threshold, lr_decay_factor;
  // inputs
  const int32_t* ids;          // [Bl]
  const double* scal;          // [2] step scalars {gamma_t, eps_t}
  float* diag;                 // [B]
  // dataset-sized tables (fp64 SoA)
  double* u1_tab; double* u2_tab;
  double* tau1_tab; double* tau2_tab;
  double* m1_tab; double* v1_tab; long long* s1_tab;
  double* m2_tab; double* v2_tab; long long* s2_tab;
  TauState* tau_state;
  // pass-1 products
  float2* rowstat_R; float2* rowstat_C;   // [Bl]
  float2* partial_R; float2* partial_C;   // [Bl][n_jt*4]
  const float2* col_partial;             // fused pass 1 (K = 1): segment-C stats [B/32][col_slots][32]
  int col_slots;                         // 0: segment-C stats are row partials in partial_C
  unsigned long long* clamps;
  float* bounds;                         // this rank's slot {max |E1|^2, max |E2|^2, max kappa} (atomicMax on float bits)
  // per-local-anchor fp64 state of the step
  double* t_loc1; double* t_loc2;
  double* sum1; double* dx1; double* sum2; double* dx2;
  double* g1; double* g2; double* u1; double* u2;
  double* term_a; double* term_b; double* term_loss;
  double* gt1; double* gt2;              // v2 tau gradients, contiguous [gt1 | gt2] (send)
  // packed per-rank payload (all-gathered at K > 1; recv == send at K == 1):
  //   [u1 | u2 | t1 | t2 | id | gt1 | gt2] x Bl, then nblk x {G_tau term a, term b, loss}
  // so one all-gather carries the per-sample scalars, the v2 per-index tau gradients and the
  // per-block partial sums of G_tau and the loss (no separate all-reduce / gather)
  double* send;                          // [pstride]
  const double* recv;                    // [K][pstride]
  int pstride, nblk;
  // pass-2 parameters
  // per-anchor exponent parameters y = s*kappa + beta and weights coef (SoA, [n_jt*256])
  float* kap1; float* bet1; float* coef1;   // track 1: kappa = log2e/t1, coef = w1/t1
  float* kap2; float* bet2; float* coef2;   // track 2: kappa = log2e/t2, coef = w2/t2
  float* fac1; float* fac2;                 // coef * 2^beta (factorized pass 2, one shared temperature)
  float* rcoef;                          // [Bl]
  double* red;                           // [2] local G_tau, loss numerator (all-reduced)
  double* blockpart;                     // [nblk][3] per-block partial sums (send + 7 Bl)
  int n_blockpart;                       // blocks of the kernel that wrote blockpart
  int* err;
  StepResult* result;
  float gscale;                          // c = 1 / (Bl (B-1)), engine.cpp:84-85
  long long* dbg;                        // FC_PROFILE builds: per-block globaltimer stamps of fc_anchor_kernel
  int prep_row0, prep_rows;              // rows of the prep kernel (all of G, or this rank's L before the gather)
  int weights_replica_only;              // fc_weights_kernel: only the u replica update (parameters arrived)
  unsigned long long* step_tag;          // the step's sequence number (prep writes it; pass 1's id set uses it)
};

__global__ void fc_prep_kernel(const __nv_bfloat16* __restrict__ e1, const __nv_bfloat16* __restrict__ e2,
                               StepArgs a, double gamma, double eps, unsigned long long seq);
// device-side error codes (first failure wins), the fc_status values of fastclip_b200.h
constexpr int kErrShape = 2, kErrOwnership = 5, kErrNumeric = 9;
__global__ void fc_weights_kernel(StepArgs a);
__global__ void fc_anchor_kernel(StepArgs a);
__global__ void fc_delay_kernel(long long ns);
__global__ void fc_rs_mask_kernel(StepArgs a);
__global__ void fc_axpy2_kernel(float* y1, float* y2, const float* x1, const float* x2, long long n, float c);
__global__ void fc_reduce_kernel(StepArgs a);
__global__ void fc_indiv_update_kernel(StepArgs a);
__global__ void fc_rows_kernel(const __nv_bfloat16* __restrict__ e1, const __nv_bfloat16* __restrict__ e2, int B,
                               int d, int lo, int cnt, const double* __restrict__ t1, const double* __restrict__ t2,
                               float2* rowstat_R, float2* rowstat_C, float* bounds, float* diag);
__global__ void fc_pair_params_kernel(const float* __restrict__ diag, const double* __restrict__ w1,
                                      const double* __restrict__ w2, const double* __restrict__ t1,
                                      const double* __restrict__ t2, int B, float* kap1, float* bet1, float* coef1,
                                      float* fac1, float* kap2, float* bet2, float* coef2, float* fac2,
                                      float* bounds);
__global__ void fc_rcoef_kernel(const float2* __restrict__ pR, const float2* __restrict__ pC, int nparts, int cnt,
                                int lo, const double* __restrict__ w1, const double* __restrict__ w2,
                                const double* __restrict__ t1, const double* __restrict__ t2, float* rcoef);
__global__ void fc_gsum_kernel(const float2* __restrict__ pR, const float2* __restrict__ pC, int nparts, int cnt,
                               int B, const float2* __restrict__ rsR, const float2* __restrict__ rsC,
                               const double* __restrict__ t1, const double* __restrict__ t2, double* g1, double* g2,
                               double* ds1, double* ds2);

}  // namespace fc
