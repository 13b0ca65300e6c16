/*
 * fastclip_b200.h -- C ABI of the B200-native FastCLIP loss step.
 *
 * Drop-in boundary for the per-worker loss step of the reference trainer
 * (proj/core/src/trainer.cpp:427-589). The reference has no FFI: the step is a sequence of
 * C++ namespace calls (engine::g_values, UTable::update/snapshot, engine::weights_*,
 * engine::embedding_cotangents, engine::grad_tau_*, opt::temperature_step and the fabric
 * collectives). Each entry point below cites the reference interface it replaces.
 *
 * Conventions: plain pointers and sizes only; embeddings are bf16 row-major [rows x dim]
 * (the reference's L2-normalised E rows, engine.hpp:45-53), gradients fp32, tables fp64
 * (state.hpp:37-122). Device pointers are marked (device); one context per rank, not
 * thread-safe, stream-ordered. Status codes map 1:1 onto errors.hpp:10-60; no C++
 * exception crosses this boundary; fc_last_error() returns the message of the last failure.
 */
#ifndef FASTCLIP_B200_H
#define FASTCLIP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes (errors.hpp:10-60). */
typedef enum {
  FC_OK = 0,
  FC_ERR_CONFIG = 1,             /* ConfigError */
  FC_ERR_SHAPE = 2,              /* ShapeError */
  FC_ERR_DEGENERATE_BATCH = 3,   /* DegenerateBatchError (B < 2) */
  FC_ERR_DOMAIN = 4,             /* std::domain_error (tau <= 0, eps < 0, gamma outside (0,1]) */
  FC_ERR_OWNERSHIP = 5,          /* OwnershipViolation (duplicate ids in one step) */
  FC_ERR_STALENESS = 6,          /* StalenessError */
  FC_ERR_COLLECTIVE_SHAPE = 7,   /* CollectiveShapeError */
  FC_ERR_COLLECTIVE_ABORTED = 8, /* CollectiveAborted (NCCL async error on a peer) */
  FC_ERR_NUMERIC = 9,            /* NumericError (non-finite tau gradient) */
  FC_ERR_IO = 10,                /* IoError (table upload/download size mismatch) */
  FC_ERR_CUDA = 11,              /* CUDA runtime / driver failure */
  FC_ERR_NCCL = 12,              /* NCCL failure */
  FC_ERR_UNSUPPORTED = 13        /* shape outside the kernels' contract (e.g. dim % 8 != 0) */
} fc_status;

/* Variants in the reference's enum order (trainer.hpp:145-153). */
typedef enum {
  FC_OPENCLIP_MBCL = 0,
  FC_SOGCLR = 1,
  FC_ISOGCLR = 2,
  FC_FASTCLIP_V0 = 3,
  FC_FASTCLIP_V1 = 4,
  FC_FASTCLIP_V2 = 5,
  FC_FASTCLIP_V3 = 6
} fc_variant;

/* Fully resolved step configuration: AlgoConfig (trainer.hpp:164-187) restricted to the
 * loss step + TempConfig (state.hpp:81-89) + AdamConfig (optimizers.hpp:10-15). */
typedef struct {
  int32_t variant;            /* fc_variant */
  int64_t n_train;            /* N: u/tau table size and the v2 1/N prefactor */
  int32_t dim;                /* d (multiple of 8) */
  int32_t local_batch;        /* Bl = global batch / world (trainer.hpp:186) */
  int32_t world;              /* K ranks (one GPU each) */
  int32_t rank;               /* this rank, owns global rows [rank*Bl, (rank+1)*Bl) */
  double tau_init;            /* temperature.init */
  double tau0;                /* projection floor */
  double rho;                 /* margin (v2/v3) */
  double tau_lr;              /* temperature.lr */
  double beta1, beta2, adam_eps;
  int32_t lr_decay_enabled;   /* TauLrLatch (schedules.hpp:52-59) */
  double lr_decay_threshold;
  double lr_decay_factor;
  int32_t scale_by_tau;       /* loss.scale_by_tau resolved (trainer.cpp:184-194) */
  int32_t device;             /* CUDA device ordinal */
  uint8_t nccl_id[128];       /* ncclUniqueId from rank 0 (fc_nccl_unique_id), world > 1 */
  int32_t reduction;          /* fabric.reduction (trainer.cpp:85-95): 0 fastclip (all-gather u, each rank
                                 computes both loss terms), 1 openclip_rs (local weights only, the contrast
                                 cotangents of the other ranks' anchors reduce-scattered; world > 1) */
} fc_config;

/* Inputs of one step (trainer.cpp:419-425 outputs + step scalars). */
typedef struct {
  const void* e1;             /* (device) bf16 [Bl x dim]: local image embeddings */
  const void* e2;             /* (device) bf16 [Bl x dim]: local text embeddings */
  const int32_t* ids;         /* (device) int32 [Bl]: distinct dataset indices of the local batch */
  double gamma;               /* inner LR gamma_t (GammaSchedule::at, schedules.cpp:25-31) */
  double eps;                 /* epsilon_t (EpsilonSchedule::at, schedules.cpp:62-65) */
} fc_step_in;

/* Outputs of one step. */
typedef struct {
  float* de1;                 /* (device) fp32 [Bl x dim]: engine::Cotangents::d_e1 */
  float* de2;                 /* (device) fp32 [Bl x dim]: engine::Cotangents::d_e2 */
} fc_step_out;

/* Scalars of the last step (read after the step's stream work completes). */
typedef struct {
  double loss;                /* exact batch loss at tau^t (losses.cpp:126-180 per variant) */
  double gtau;                /* all-reduced G_tau (trainer.cpp:572); 0 for v1/v2 */
  double tau;                 /* global tau after the step (temperature_step) */
  uint64_t exp_clamps;        /* safe_exp clamps among the local g evaluations */
  int32_t latched;            /* TauLrLatch state after the step */
} fc_step_scalars;

/* resolve_algo_config's temperature / loss defaults for `variant` (trainer.cpp:139-194,
 * config.cpp:36-60). Leaves dim/local_batch/world/rank/device zero. */
int fc_config_defaults(int32_t variant, int64_t n_train, fc_config* out);

/* GammaSchedule::at (schedules.cpp:25-31), cosine or constant kind. */
double fc_gamma_at(int32_t cosine, double constant, double gamma_min, int64_t decay_epochs,
                   int64_t iters_per_epoch, int64_t t);
/* EpsilonSchedule::at (schedules.cpp:62-65); switch_epoch < 0 = never. */
double fc_epsilon_at(double initial, double late, int64_t switch_epoch, int64_t epoch);

/* New NCCL unique id (rank 0), to be broadcast to the other ranks out of band. */
int fc_nccl_unique_id(uint8_t out[128]);

/* Creates a rank context: device u/tau tables (u = 0, tau = init: state.cpp:42-43,105-110),
 * workspaces, streams and (world > 1) the NCCL communicator. */
int fc_create(const fc_config* cfg, void** ctx);
int fc_destroy(void* ctx);

/* One loss step: trainer.cpp:427-589 for this rank. Enqueued on `stream` (cudaStream_t,
 * NULL = legacy default); asynchronous. Replaces, in order: g_values (engine.cpp:151-176),
 * UTable::update/snapshot (state.cpp:45-71), the u/tau all-gathers (trainer.cpp:459-487),
 * weights_* (engine.cpp:37-75), embedding_cotangents (engine.cpp:77-121), grad_tau_*
 * (engine.cpp:208-266), all_reduce_mean_scalar (fabric.cpp:210-212) and
 * temperature_step / IndividualTemp::update (optimizers.cpp:77-83, state.cpp:124-131). */
int fc_loss_step(void* ctx, const fc_step_in* in, fc_step_out* out, void* stream);

/* Waits for the last step and returns its scalars. Failures the device detects during a step
 * are returned here and stay set for the context (the reference throws and the run ends):
 * FC_ERR_SHAPE for an id outside [0, n_train) (state.cpp:46; the table is never written at
 * such an id), FC_ERR_NUMERIC for a non-finite tau gradient (optimizers.cpp:67), FC_ERR_NCCL
 * when a peer all-gather handshake times out (a rank stopped stepping). */
int fc_step_scalars_get(void* ctx, fc_step_scalars* out);

/* Per-anchor views of the last step for the local rows (host fp64 [Bl] each, may be NULL):
 * g1/g2 (engine.cpp:151-176), u1/u2 snapshot (state.cpp:57-71; g for MBCL), t1/t2 = tau^t. */
int fc_local_views(void* ctx, double* g1, double* g2, double* u1, double* u2, double* t1, double* t2);

/* Table checkpoint hooks (UTable / IndividualTemp SoA, state.cpp:73-95,133-162): host fp64
 * [n_train] arrays; tau/m/v/step arrays only for individual-temperature variants (else NULL). */
int fc_table_download(void* ctx, double* u1, double* u2, double* tau1, double* tau2, double* m1,
                      double* v1, int64_t* s1, double* m2, double* v2, int64_t* s2);
int fc_table_upload(void* ctx, const double* u1, const double* u2, const double* tau1,
                    const double* tau2, const double* m1, const double* v1, const int64_t* s1,
                    const double* m2, const double* v2, const int64_t* s2);
/* Global tau replica state (Replica::tau, tau_adam, latch; trainer.cpp:245-254). */
int fc_tau_state_get(void* ctx, double* tau, double* m, double* v, int64_t* step, int32_t* latched);
int fc_tau_state_set(void* ctx, double tau, double m, double v, int64_t step, int32_t latched);

/* Per-phase CUDA-event timing of the step (off by default; slots = 0 turns it off). Phases:
 * 0 embedding all-gather, 1 diag + tau^t row parameters, 2 pass-1 similarity statistics,
 * 3 tables/weights/tau update (+ scalar collectives), 4 pass-2 Q tiles, 5 gradient GEMM.
 * Steps cycle through `slots` event sets, so timed steps need no host synchronisation;
 * fc_phase_times(slot) waits for that set (slot < 0: the last step) and returns ms per phase. */
int fc_set_phase_timing(void* ctx, int32_t slots);
int fc_phase_times(void* ctx, int32_t slot, float* ms, int32_t n);

/* Number of CUDA kernels fc_loss_step enqueues per step (launch accounting for the bench). */
int fc_kernels_per_step(void* ctx);

/* Raw S = A B^T through the pass-1 tcgen05 tile kernel (diagnostics / kernel unit tests):
 * a [rows x dim], b [cols x dim] bf16 (device), out fp32 [rows x cols] (device). */
int fc_debug_similarity(const void* a, const void* b, int32_t rows, int32_t cols, int32_t dim,
                        float* out, void* stream);

/* Per-function entry point for parity / a stateless caller: engine::g_values
 * (engine.cpp:151-176) and, when dsum1/dsum2 are non-NULL, engine::dtau_sums (engine.cpp:182-204)
 * for the local slice [local_begin, local_begin + local_count) of a global batch, computed by the
 * step's tcgen05 pass-1 kernel. e1g/e2g: (device) bf16 [batch x dim]; t1/t2_local: (device) fp64
 * [local_count] (tau^t of the local anchors; dtau_sums' t is the same per-anchor value,
 * engine.cpp:198-199); outputs (device) fp64 [local_count]; clamps: (device, may be NULL) the
 * number of safe_exp clamps among the evaluated exponentials (losses.cpp:10). Asynchronous on
 * `stream`. Errors: FC_ERR_DEGENERATE_BATCH (batch < 2), FC_ERR_SHAPE (slice outside the batch,
 * engine.cpp:11-19), FC_ERR_UNSUPPORTED (dim % 8 != 0). */
int fc_g_values(const void* e1g, const void* e2g, int32_t batch, int32_t dim, const double* t1_local,
                const double* t2_local, int32_t local_begin, int32_t local_count, double* g1, double* g2,
                double* dsum1, double* dsum2, uint64_t* clamps, void* stream);

/* Per-function entry point: engine::embedding_cotangents (engine.cpp:77-121) for the local
 * slice [local_begin, local_begin + local_count) of a global batch with the caller's PairWeights
 * (engine.hpp:29-32) over G: w1, w2, t1, t2 (device) fp64 [batch]. e1g/e2g: (device) bf16
 * [batch x dim]; de1/de2: (device) fp32 [local_count x dim], overwritten (scale 1/(local_count
 * (batch-1)), engine.cpp:84-85). Runs the step's pass-1, pass-2 and gradient-GEMM kernels;
 * asynchronous on `stream`. Errors as fc_g_values. */
int fc_embedding_cotangents(const void* e1g, const void* e2g, int32_t batch, int32_t dim, const double* w1,
                            const double* w2, const double* t1, const double* t2, int32_t local_begin,
                            int32_t local_count, float* de1, float* de2, void* stream);

/* opt::temperature_step (optimizers.cpp:77-83): Adam with weight decay 0 (bias correction with
 * step + 1, then ++step; optimizers.cpp:65-75) and the projection max(tau, tau0). Host scalar;
 * FC_ERR_NUMERIC for a non-finite gradient (optimizers.cpp:67). */
int fc_temperature_step(double* m, double* v, int64_t* step, double tau, double grad, double lr, double beta1,
                        double beta2, double eps, double tau0, double* tau_out);

/* UTable::update + snapshot (state.cpp:45-71) on caller-owned device tables u1/u2 [n_train]:
 * u <- (1 - gamma) u + gamma g at ids[0..count) (distinct), post-update values into
 * u1_out/u2_out [count] (may be NULL). FC_ERR_DOMAIN for gamma outside (0,1] (state.cpp:50);
 * a device-side ShapeError (id outside [0, n_train), state.cpp:46) or domain_error (g < 0,
 * state.cpp:51) is written to *status (device int32, may be NULL) and that entry is skipped. */
int fc_table_update(double* u1, double* u2, int64_t n_train, const int32_t* ids, const double* g1, const double* g2,
                    int32_t count, double gamma, double* u1_out, double* u2_out, int32_t* status, void* stream);

/* engine::grad_tau_* for one worker's local anchors from their dtau sums (fc_g_values) and u
 * snapshot (for MBCL, u = g): v0 grad_tau_unscaled (engine.cpp:208-224), v3 grad_tau_margin
 * (:226-238) and MBCL (:261-266) write G_tau,k to gtau[0] (before the mean all-reduce,
 * trainer.cpp:572); v2 / iSogCLR grad_tau_individual (:240-259) write gt1/gt2 [count] (needs
 * t1/t2 and n_train). All pointers (device) fp64; fixed-order reduction. FC_ERR_CONFIG for the
 * constant-tau variants (no tau gradient). */
int fc_grad_tau(int32_t variant, int32_t count, int64_t batch, const double* u1, const double* u2, const double* dsum1,
                const double* dsum2, const double* t1, const double* t2, double eps, double rho, double tau,
                int64_t n_train, double* gtau, double* gt1, double* gt2, void* stream);

/* ---- on-disk state in the reference's binary formats ---- */

/* UTable::write (state.cpp:73-76: int64 n + n doubles per track, u1 then u2) followed, for the
 * individual-temperature variants, by IndividualTemp::write (state.cpp:133-144: tau1, tau2, tau0,
 * then the {m, v, step} ScalarAdam records of both tracks): the context's device tables to `path`.
 * Synchronises the device. FC_ERR_IO when the file cannot be written. */
int fc_table_write(void* ctx, const char* path);
/* UTable::read / IndividualTemp::read (state.cpp:87-95, :146-162) into the device tables.
 * FC_ERR_IO on a truncated stream or differing track lengths (IoError), FC_ERR_SHAPE when the
 * table size differs from n_train (UTable::load, state.cpp:78-81). */
int fc_table_read(void* ctx, const char* path);

/* The model part of an FCK1 checkpoint (io::Checkpoint, checkpoint.hpp:16-40): the loss step
 * owns the temperature, its Adam state and latch, and the tables; the caller owns the rest. */
typedef struct {
  uint64_t seed;
  int64_t next_epoch;
  int64_t global_step;
  int32_t image_shape[4];     /* TowerShape: kind (0 linear, 1 mlp), d_in, d_hidden, d_out */
  int32_t text_shape[4];
  int64_t n_params;           /* length of params / opt_m / opt_v */
  double* params;             /* host [n_params] (read: filled when non-NULL and n_params matches) */
  double* opt_m;
  double* opt_v;
  int64_t opt_step;
} fc_model_state;

/* write_checkpoint (checkpoint.cpp:57-82): magic "FCK1", the model part (NULL: empty model), then
 * this context's tau, tau-Adam {m, v, step}, latch, u1, u2 and the IndividualTemp record. */
int fc_checkpoint_write(void* ctx, const char* path, const fc_model_state* model);
/* read_checkpoint (checkpoint.cpp:84-114) for a resume: restores tau / tau-Adam / latch / tables into
 * the context and returns the model part in *model (may be NULL). FC_ERR_IO on a bad magic or a
 * truncated file, FC_ERR_CONFIG when the IndividualTemp record does not match the variant. */
int fc_checkpoint_read(void* ctx, const char* path, fc_model_state* model);

/* ---- the model-side step after the loss step (§8(f) row 1), fp64 device arrays ---- */

/* TwoTowerModel::forward (encoder.cpp:98-134) of one tower: kind 0 linear (theta = [W (d_out x
 * d_in) | b]), kind 1 tanh-MLP (theta = [W1 | b1 | W2 | b2]); x [rows x d_in]; h [rows x d_hidden]
 * (mlp, else NULL), z / e [rows x d_out], znorm [rows]; e_bf16 (may be NULL): e rounded to bf16, the
 * loss step's input. *status (device int32) gets FC_ERR_NUMERIC for a row with |z| < 1e-12. */
int fc_tower_forward(int32_t kind, int32_t rows, int32_t d_in, int32_t d_hidden, int32_t d_out, const double* theta,
                     const double* x, double* h, double* z, double* e, double* znorm, uint16_t* e_bf16,
                     int32_t* status, void* stream);
/* TwoTowerModel::vjp (encoder.cpp:136-177): the loss step's dE (fp32 [rows x d_out]) through the
 * normalisation Jacobian, cot_z = (cot - e (e . cot)) / |z|, into the tower's parameter gradient
 * (accumulated into grad, the tower's slice of the flat gradient; assemble_packet, engine.cpp:268-276). */
int fc_tower_vjp(int32_t kind, int32_t rows, int32_t d_in, int32_t d_hidden, int32_t d_out, const double* theta,
                 const double* x, const double* h, const double* e, const double* znorm, const float* cot,
                 double* grad, void* stream);
/* all_reduce_mean "grad-reduce" (trainer.cpp:540-546, fabric.cpp:204-208) of a flat gradient over
 * the context's ranks (in place; a no-op at world 1). */
int fc_grad_allreduce_mean(void* ctx, double* grad, int64_t n, void* stream);
/* opt::adamw_step (optimizers.cpp:33-41) on a flat parameter vector; *step is the host step counter
 * (bias corrections 1 - beta^(step+1), then ++step). A non-finite gradient sets *status (device
 * int32) to FC_ERR_NUMERIC and leaves theta / m / v unchanged (check_shapes, optimizers.cpp:13). */
int fc_adamw_step(int64_t n, double* theta, double* m, double* v, int64_t* step, const double* grad, double lr,
                  double beta1, double beta2, double eps, double weight_decay, int32_t* status, void* stream);
/* opt::lamb_step (optimizers.cpp:43-63): per-layer trust ratios over the segments
 * [seg_off[k], seg_off[k] + seg_len[k]) (host arrays), ratio 1 for a zero denominator or with
 * force_alpha_one. Synchronises `stream` before returning. */
int fc_lamb_step(int64_t n, double* theta, double* m, double* v, int64_t* step, const double* grad, double lr,
                 double beta1, double beta2, double eps, double weight_decay, int32_t n_seg, const int64_t* seg_off,
                 const int64_t* seg_len, int32_t force_alpha_one, int32_t* status, void* stream);
const char* fc_model_last_error(void);

/* ---- the step before the hot path: index stream and synthetic inputs (§8(f) row 4) ---- */

/* BatchPlan (trainer.cpp:206-241) over the reference's RNG streams (rng.hpp:14-65: splitmix64
 * stream ids, std::mt19937_64, rejection `below`, descending Fisher-Yates): epoch permutations and
 * per-worker contiguous slices identical to the reference's. FC_ERR_CONFIG when the global batch
 * does not divide n_train (trainer.cpp:208-213) or the world does not divide the batch. */
int fc_batch_plan_create(int64_t n_train, int32_t global_batch, uint64_t seed, void** plan);
int fc_batch_plan_destroy(void* plan);
int64_t fc_batch_plan_iters_per_epoch(void* plan);
int fc_batch_plan_permutation(void* plan, int64_t epoch, int32_t* out /* [n_train] */);
int fc_batch_plan_local(void* plan, int64_t epoch, int64_t iter, int32_t worker, int32_t world,
                        int32_t* out /* [global_batch / world] */);
const char* fc_plan_last_error(void);
/* SURVEY.md §8(d) synthetic inputs from the seed's rng.hpp streams: unit-norm E1 rows and
 * E2 = normalize(E1 + sigma N(0, I)), rounded to bf16 (host arrays [rows x dim] of bf16 bits); and
 * `count` distinct ids in [0, n) by a partial Fisher-Yates. */
int fc_synthetic_embeddings(uint64_t seed, int32_t rows, int32_t dim, double sigma, uint16_t* e1, uint16_t* e2);
int fc_synthetic_ids(uint64_t seed, int32_t count, int64_t n, int32_t* ids);
/* a warm u table: log10 u ~ U[-8, 0] (the paper's u percentiles), host [n] */
int fc_synthetic_warm_u(uint64_t seed, int64_t n, double* out);

/* CommLedger (fabric.hpp:34-58) of the context's steps: one entry per collective phase of the
 * reference's fabric ("feature-gather", "u-gather", "tau-gather", "tau-reduce", "rs-grad") with its
 * primitive (0 all_gather, 1 all_reduce, 2 reduce_scatter), the reference's wire elements
 * (fabric.cpp:18-28 ring costs, accumulated over steps) and the bytes this rank actually stored to
 * its peers for that phase (NVLink peer stores or NCCL payloads; the packed payload gather is
 * split by its fields, and "replica-sync" carries what only the per-GPU table replicas need).
 * Returns the number of entries written (<= max). */
typedef struct {
  char phase[24];
  int32_t primitive;
  int32_t world;
  uint64_t elements;
  uint64_t bytes;
} fc_ledger_entry;
int fc_comm_ledger(void* ctx, fc_ledger_entry* out, int32_t max);
int fc_comm_ledger_reset(void* ctx);

const char* fc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* FASTCLIP_B200_H */
