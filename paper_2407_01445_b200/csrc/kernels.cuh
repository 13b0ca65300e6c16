// kernels.cuh -- parameter blocks and launchers of the FastCLIP B200 kernels.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

namespace fc {

// globaltimer / cycle stamps of the profiling builds (FC_PROFILE=1 python -m paper_2407_01445_b200.build);
// the shipped library compiles every stamp out
#ifdef FC_PROFILE
constexpr bool kProfStamps = true;
#else
constexpr bool kProfStamps = false;
#endif

// ---- tiling shared by the two tcgen05 kernels (CTA pair = cluster of 2, cta_group::2) ----
constexpr int kPairM = 256;      // rows per pair tile (128 per CTA)
constexpr int kCtaM = 128;       // TMEM lanes / rows per CTA
constexpr int kPairN = 256;      // columns per pair tile (UMMA N)
constexpr int kBlockK = 64;      // bf16 per 128-byte swizzle atom
constexpr int kStageBytesA = kCtaM * kBlockK * 2;        // 16 KB
constexpr int kStageBytesB = (kPairN / 2) * kBlockK * 2;  // 16 KB (own half of N)
// similarity kernel: A (the anchor rows) stays resident for up to 8 K blocks (d <= 512;
// larger d streams A in 512-wide chunks through the same slots), B streams through a ring.
constexpr int kSimASlots = 8;
constexpr int kSimStagesStats = 5;   // B ring depth, statistics pass
constexpr int kSimStagesQ = 3;       // B ring depth, Q pass (smem goes to the Q store staging)
constexpr int kSimStageOutQ = 32 * 64;   // per epilogue warp: 32 rows x 32 bf16 (64-byte swizzled rows)
constexpr int kSimEpiWarps = 16;   // 4 per TMEM lane quarter, 64 columns each
constexpr int kSimThreads = (2 + kSimEpiWarps) * 32;
constexpr int kSimPSlots = 3;      // column-parameter slots (Q pass): kappa, beta, coef, fac x 256
constexpr int kSimPSlotBytes = 4 * kPairN * 4;   // kappa, beta, coef, fac
// STATS / FUSED / RAW: the parameter region doubles as the fused pass's column-sum exchange,
// [tile parity][column group][chunk][lane quarter][32] float2
constexpr int kSimRedBytes = 2 * 2 * 4 * 4 * 32 * 8;
constexpr int kSimParRedBytes = kSimRedBytes > kSimPSlots * kSimPSlotBytes ? kSimRedBytes : kSimPSlots * kSimPSlotBytes;
constexpr int kSimSmemStats = kSimASlots * kStageBytesA + kSimStagesStats * kStageBytesB + kSimParRedBytes;
constexpr int kSimSmemQ = kSimASlots * kStageBytesA + kSimStagesQ * kStageBytesB + kSimPSlots * kSimPSlotBytes +
                          kSimEpiWarps * kSimStageOutQ;
constexpr int kSimSmemBytes = (kSimSmemStats > kSimSmemQ ? kSimSmemStats : kSimSmemQ) + 1024 + 512;
// gradient GEMM: A (Q') and B (E) both stream; pair tile 256 x 512 (two N = 256 accumulators).
constexpr int kMaxGemmClusters = 160;
constexpr int kGemmN = 2 * kPairN;
constexpr int kGemmStages = 4;
constexpr int kGemmStageBytesB = 2 * kStageBytesB;   // own 128 columns of both N halves
constexpr int kGemmEpiWarps = 8;                     // 2 per TMEM lane quarter, 256 columns each
constexpr int kGemmThreads = (2 + kGemmEpiWarps) * 32;
constexpr int kGemmStageOut = 32 * 32 * 4;   // per epilogue warp: 32 rows x 32 fp32 (128-byte swizzled rows)
constexpr int kGemmSmemBytes = kGemmStages * (kStageBytesA + kGemmStageBytesB) + kGemmEpiWarps * kGemmStageOut +
                               1024 /*align*/ + 256 /*barriers*/;

// ---- similarity-tile kernel (pass 1: row statistics; pass 2: Q tiles) ----
// One "segment" is an S block S' = A B^T with A = E_rows[a_row0 .. a_row0+rows) and
// B = E_cols[0 .. cols). Segment R: (E1[L], E2[G]); segment C: (E2[L], E1[G]) so that the
// column statistics / transposed Q of S are row quantities of S'.
struct SimSeg {
  int rows;                 // local anchors in this segment
  int a_row0;               // global index of local row 0 (diagonal masking)
  int cols;                 // contrast set size (global batch B)
  const float2* row_stat;   // STATS: [rows] {kappa_i = log2(e)/t_i, beta_i = -S_ii kappa_i}
  const float2* col_stat;   // FUSED: [cols] {kappa_j, beta_j} of the column anchors (segment C)
  float2* partial;          // STATS: [rows][n_jt*4] {sum e, sum y e} per column quarter
  // Q: exponent y = s*kappa + beta (= (s - S_aa) log2(e)/t_a), weight coef (SoA, fp32)
  const float* row_kappa; const float* row_beta; const float* row_coef;   // [rows]
  const float* col_kappa; const float* col_beta; const float* col_coef;   // [n_jt*256], zero padded
  // Q, global temperature: fac_a = coef_a 2^beta_a, so Q'_ij = 2^(s kappa) (fac_i + fac_j)
  const float* row_fac; const float* col_fac;
  __nv_bfloat16* q;         // Q: [rows][ldq]
};
struct SimParams {
  SimSeg seg[2];
  int nseg;
  int d;
  int ldq;
  int n_jt;
  int n_rb[2];
  int n_items;
  unsigned long long* clamps;  // STATS: exponent clamps (safe_exp, losses.cpp:22-28)
  const float* bounds;         // [n_bounds][4] {max |E1_i|^2, max |E2_j|^2, max kappa}: one slot per rank,
  int n_bounds;                // the maxima over G are the max over the slots (clamp-free fast paths)
  int q_factor;                // Q: one shared temperature -> factorized single-exponential fast path
  int split_tail;              // leftover tiles (T mod pairs) run as 256 x 128 halves on twice the pairs
  // FUSED: column statistics {sum e, sum y e} per (row slot = one CTA of a pair row block,
  // column), laid out [cols / 32][n_slots][32] with n_slots = 2 per pair row block (the CTA's
  // four 32-row warp sums are added in shared memory); fuse_fast enables the one-exponential path
  float2* col_partial;
  int n_slots;
  int fuse_fast;
  // pass 1 also zeroes the step's gradient outputs (the GEMM reduce-adds every stream-K unit
  // into them): the epilogue warps do it while the first tiles' MMAs run
  float4* zero0;
  float4* zero1;
  long long zero_n4;
  // duplicate-id check, run by the epilogue threads before their first tile: an open-addressing set
  // of the rank's ids with slots tagged by the step's sequence number (*step_tag, written by
  // prep), so nothing is cleared between steps; a repeat sets *err = FC_ERR_OWNERSHIP before
  // the per-anchor kernel (which skips every table write then) starts
  const int* ids;
  int n_ids;
  unsigned long long* idset;
  int idset_mask;                      // slots - 1 (power of two >= 2 n_ids)
  const unsigned long long* step_tag;
  int* err;
  // K > 1: a pass overlapped with a gather; each pair runs its share of the own column tiles
  // (tiles [jt_lo, jt_lo + n_loc), wholly inside this rank's slice) first, then its share of
  // the remote ones. local_first 1 (pass 1 beside the embedding gather): A and the own tiles are
  // read from the caller's buffers (mapA*, mapQo0 / mapQo1 slots, rows from col_lo), a remote
  // tile from the gathered buffers once the producer saw the flag of each rank whose rows it
  // holds (src_flag[k] >= *step_tag). local_first 2 (pass 2 beside the payload gather): the
  // operands are all gathered already; a remote tile's column parameters wait for the flags.
  int local_first;
  int jt_lo, n_loc;
  int col_lo;                  // first global row of the caller's slice (also subtracted from A rows)
  int rows_per_src;            // rows of G per rank
  const unsigned long long* src_flag;
  const unsigned long long* abort_flag;
  long long timeout_ns;        // no flag within this long: FC_ERR_COLLECTIVE_ABORTED, stop waiting
  int exact_bounds;            // STATS: per-chunk clamp check from the tile values (no norm bounds)
  long long* dbg_out;          // FC_PROFILE builds: per-pair MMA-warp / epilogue counters, per-CTA stamps
};

// ---- weighted-gradient GEMM: out = scale * (Q' X - r o X_local) ----
struct GemmSeg {
  int a_mn_major;            // 1: A = Q'^T read through an MN-major operand (K = 1 shares Q)
  int rows;                  // local anchors
  int x_row0;                // global index of local row 0 (for the r o X_local term)
  int x_krow0;               // first row of X the K index maps to (0; rank * Bl for the reduce-scatter partials)
  const float* r;            // [rows], or NULL: no local term
  const __nv_bfloat16* x;    // [B][d] row-major (the B operand, read for the r term)
  float* out;                // [rows][d], zeroed before the GEMM (reduce-add target)
};
struct GemmParams {
  GemmSeg seg[2];
  int nseg;
  int d;
  int n_mb[2];
  int n_nb;
  int n_tiles;       // sum over segments of n_mb * n_nb (pair tiles: 256 x 512)
  // stream-K partition: pair c runs units [unit_lo[c], unit_lo[c+1]) of the (tile, k-block)
  // sequence; the host balances k-blocks + per-unit epilogue cost (a unit boundary costs one
  // accumulator drain), so pairs with two units get fewer k-blocks
  int unit_lo[kMaxGemmClusters + 1];
  int kb_total;      // K blocks of 64 over ldq
  float scale;       // 1 / (Bl (B-1)), engine.cpp:84-85
  float* reset_at_exit; // 4 * n_reset floats zeroed when the GEMM (the step's last kernel) retires: the
  int n_reset;          // next step's norm / kappa bounds start from 0 without a memset node
  long long* dbg_out;   // FC_PROFILE builds: [cta][16] MMA / epilogue counters, globaltimer stamps
};

// kSimFused (K = 1): one S tile gives both the row statistics (segment R) and the column
// statistics (segment C = S^T), so pass 1 multiplies S once instead of twice.
// ---- NVLink peer all-gather (K > 1): this rank's slices into every rank's buffer + flags ----
constexpr int kMaxPeers = 8;
constexpr int kMaxGatherSrc = 10;
struct PeerGather {
  const uint8_t* src[kMaxGatherSrc];            // this rank's slices
  uint8_t* dst[kMaxGatherSrc][kMaxPeers];       // every rank's destination (peer-mapped), slice at rank*bytes[t]
  size_t bytes[kMaxGatherSrc];                  // bytes per slice (multiples of 16)
  int n_src;
  int world, rank;
  unsigned long long seq;             // per-step sequence number (updated in the replayed graph)
  unsigned long long* peer_flag[kMaxPeers];   // rank k's flag array for this gather (peer-mapped)
  unsigned long long* my_flag;        // local flag array [world]
  unsigned* ticket;                   // local grid-completion ticket
  int* err;
  long long* dbg;                     // FC_PROFILE builds: globaltimer stamps {entry, stores done, flags out, peers in}
  int early_trigger;                  // release the next (programmatic) kernel at entry: it only
                                      // reads the gathered data after griddepcontrol.wait
  int wait_src;                       // programmatic launch: sources >= wait_src are written by the
                                      // preceding kernel (griddepcontrol.wait first); -1: none
  // failure propagation (fabric.cpp:228-235 poison): a rank that waits longer than timeout_ns
  // for a peer's flag stores a non-zero abort word into every rank (its own included); every
  // waiting rank polls its local abort word and leaves with FC_ERR_COLLECTIVE_ABORTED
  long long timeout_ns;
  int bulk;                           // 1: the slices go through the bulk-copy engine (thread 0 per CTA)
  unsigned long long* my_abort;
  unsigned long long* peer_abort[kMaxPeers];
};
cudaError_t launch_peer_gather(const PeerGather& g, int blocks, int threads, cudaStream_t s, bool pdl = false,
                               bool lean = false);
void* peer_gather_kernel_fn(bool lean = false);

enum SimMode { kSimStats = 0, kSimQ = 1, kSimRaw = 2, kSimFused = 3 };

cudaError_t launch_sim(int mode, const SimParams& p, const CUtensorMap* mapA, const CUtensorMap* mapB,
                       const CUtensorMap* mapQout, int grid, cudaStream_t s, float* raw_out, bool pdl = false);
cudaError_t sim_set_smem();
cudaError_t sim_attributes(int mode, cudaFuncAttributes* a);   // kSimStats / kSimQ
cudaError_t gemm_set_smem();
cudaError_t launch_gemm(bool pdl, const GemmParams& p, const CUtensorMap* mapQ, const CUtensorMap* mapX,
                        const CUtensorMap* mapOut, int grid, cudaStream_t s);

}  // namespace fc
