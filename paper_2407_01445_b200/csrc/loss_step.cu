// loss_step.cu -- host runtime of the B200 FastCLIP loss step behind the C ABI
// (include/fastclip_b200.h). One LossStep per rank: it owns the dataset-sized u/tau tables
// in HBM, the per-step workspaces, the TMA descriptors and (world > 1) an NCCL
// communicator, and enqueues the step of trainer.cpp:427-589 on a CUDA stream:
//
//   [K>1] all-gather E1, E2 (bf16)                        trainer.cpp:422-425
//   diag + tau^t row parameters                           trainer.cpp:428-434
//   pass 1: tcgen05 S tiles -> row statistics             engine.cpp:151-176, :182-204
//   table: g, UTable EMA + snapshot, packed payload       state.cpp:45-71
//   [K>1] all-gather [u1|u2|t1|t2|id] (fp64)              trainer.cpp:459-487
//   weights for the whole batch, r_i, tau-grad terms      engine.cpp:37-75, :208-266
//   [K>1] all-reduce [G_tau, loss]                        trainer.cpp:572
//   tau update (global Adam / v2 per-index Adam)          optimizers.cpp:65-83, state.cpp:124-131
//   pass 2: tcgen05 S tiles -> bf16 Q' tiles              engine.cpp:91-118 (weights)
//   tcgen05 GEMM Q' E -> dE1, dE2                         engine.cpp:77-121
#include <cuda.h>
#include <algorithm>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <nccl.h>
#include <nvtx3/nvtx3.hpp>   // header-only ranges: no-ops unless a tool injects a collector

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "../../include/fastclip_b200.h"
#include "kernels.cuh"
#include "table_kernels.cuh"

namespace {

thread_local std::string g_last_error;

struct FcError {
  int code;
  std::string msg;
};

#define FC_CUDA(call)                                                                          \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess)                                                                     \
      throw FcError{FC_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)};          \
  } while (0)
#define FC_NCCL(call)                                                                          \
  do {                                                                                         \
    ncclResult_t r_ = (call);                                                                  \
    if (r_ != ncclSuccess) throw FcError{FC_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_)}; \
  } while (0)

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    FC_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) throw FcError{FC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable"};
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2D map over a row-major [outer x inner] array with a 128-byte swizzled box (bf16 or fp32).
CUtensorMap make_map(const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes, uint32_t box_inner,
                     uint32_t box_outer, CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                     CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
  CUtensorMap m;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_bytes};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, dt, 2, const_cast<void*>(base), dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw FcError{FC_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")"};
  return m;
}

template <class T>
T* dalloc(size_t n) {
  T* p = nullptr;
  if (n == 0) n = 1;
  FC_CUDA(cudaMalloc(&p, n * sizeof(T)));
  return p;
}

int sm_count(int dev) {
  int n = 0;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

bool is_individual(int v) { return v == FC_ISOGCLR || v == FC_FASTCLIP_V2; }

// Contiguous stream-K ranges over the (tile, k-block) sequence with equal estimated cost
// per cluster: k-blocks + kDrain per unit (each unit ends in a full-tile epilogue that the
// single TMEM accumulator cannot overlap). Greedy fill against a binary-searched budget.
static void balance_stream_k(fc::GemmParams& gp, int n_clusters, int gemm_drain) {
  const long long KB = gp.kb_total, U = static_cast<long long>(gp.n_tiles) * KB;
  // cost of one unit boundary in k-blocks (measured best ~8 at K = 5120; FC_GEMM_DRAIN overrides)
  const long long kDrain = gemm_drain > 0 ? gemm_drain : std::max<long long>(1, KB / 10);
  auto fill = [&](long long budget, bool write) {
    long long u = 0;
    int c = 0;
    for (; c < n_clusters && u < U; ++c) {
      if (write) gp.unit_lo[c] = static_cast<int>(u);
      long long left = budget;
      while (u < U) {
        const long long in_tile = KB - u % KB;
        if (left <= kDrain) break;
        const long long take = std::min(in_tile, left - kDrain);
        u += take;
        left -= take + kDrain;
        if (take < in_tile) break;
      }
    }
    if (write) for (int k = c; k <= n_clusters; ++k) gp.unit_lo[k] = static_cast<int>(U);
    return u >= U;
  };
  long long lo = 1, hi = U + kDrain * (gp.n_tiles + 1);
  while (lo < hi) {   // smallest budget that covers every unit with n_clusters clusters
    const long long mid = (lo + hi) / 2;
    if (fill(mid, false)) hi = mid; else lo = mid + 1;
  }
  fill(lo, true);
  gp.unit_lo[n_clusters] = static_cast<int>(U);
}


struct LossStep {
  fc_config cfg{};
  int B = 0, Bl = 0, d = 0, K = 1, rank = 0, ldq = 0, n_jt = 0, n_sm = 148;
  bool indiv = false, track_u = true;
  ncclComm_t comm = nullptr;
  // tables
  double *u1 = nullptr, *u2 = nullptr, *tau1 = nullptr, *tau2 = nullptr, *m1 = nullptr, *v1 = nullptr,
         *m2 = nullptr, *v2 = nullptr;
  long long *s1 = nullptr, *s2 = nullptr;
  fc::TauState* tau_state = nullptr;
  // workspaces
  // gathered embeddings (K > 1), two buffers selected by the step parity: a rank may start
  // step t+1's embedding gather (its first cross-rank store) while a slower peer still reads
  // step t's rows; it cannot reach step t+2's gather before every peer has finished step t
  // (step t+1's payload gather waits for all peers, and a peer's step-(t+1) payload flag
  // follows its whole step t in stream order). The bounds slots are double-buffered alike.
  __nv_bfloat16 *e1g = nullptr, *e2g = nullptr;   // [2][B][d]
  // NVLink peer gathers (K > 1, all ranks P2P-capable; FC_PEER=0 forces the NCCL path)
  bool use_peer = false;
  int my_dev = 0;
  unsigned long long* pflags = nullptr;   // [2][kMaxPeers] local flags: E gather, payload gather; + abort word
  unsigned* ptickets = nullptr;           // [2] grid-completion tickets
  std::vector<void*> peer_maps;           // cudaIpcOpenMemHandle mappings to close
  fc::PeerGather pg_e[2]{}, pg_p[2]{};     // per step parity
  unsigned long long seq = 0;             // per-step sequence number (same on every rank)
  float* diag = nullptr;
  float2 *rowstat = nullptr, *partial = nullptr, *col_partial = nullptr;
  unsigned long long* clamps = nullptr;
  float* bounds = nullptr;   // [2][kMaxPeers][4] (parity, rank slot)
  double* f64 = nullptr;   // per-local-anchor fp64 arrays
  double *send = nullptr, *recv = nullptr, *red = nullptr;
  int nblk = 0, pstride = 0;   // payload: [u1|u2|t1|t2|id|gt1|gt2] x Bl + nblk x 3 block partials
  float* par = nullptr;   // 6 x [n_jt*256]: kap1, bet1, coef1, kap2, bet2, coef2
  float* rcoef = nullptr;
  __nv_bfloat16* q = nullptr;   // [2][Bl][ldq]
  int* err = nullptr;
  // openclip_rs (fabric.reduction = openclip_rs, K > 1): the other ranks' anchors get zero
  // pass-2 weights here; their contrast cotangents arrive reduce-scattered (trainer.cpp:492-537)
  bool rs = false;
  float* rs_part = nullptr;    // [2][B][d] fp32: for_e1, for_e2 (engine.cpp:123-144) of this rank's anchors
  float* rs_shard = nullptr;   // [2][Bl][d] fp32: the reduce-scattered sums for this rank's rows
  CUtensorMap mQtRS[2], mPart[2];
  struct LedgerRow {
    std::string phase;
    int primitive;
    unsigned long long elements, bytes;
  };
  std::vector<LedgerRow> ledger;
  void book(const char* phase, int prim, unsigned long long elements, unsigned long long bytes) {
    for (auto& r : ledger)
      if (r.phase == phase) {
        r.elements += elements;
        r.bytes += bytes;
        return;
      }
    ledger.push_back({phase, prim, elements, bytes});
  }
  long long test_delay_ns = 0;           // FC_TEST_DELAY_US (tests only, K > 1): this rank stalls after
                                         // the payload gather, before pass 2 (rank-skew stress test)
  unsigned long long* idset = nullptr;   // duplicate-id set (pass 1's non-leader MMA warps)
  int idset_slots = 0;
  unsigned long long* step_tag = nullptr;
  bool dup_check = true;                 // FC_DUP_CHECK=0: skip the duplicate-id check (A/B only)
  bool peer_bulk = false;                // FC_PEER_BULK=1: the embedding gather through the bulk-copy engine
  // K > 1 with peer memory: the embedding gather runs on its own stream beside pass 1, which
  // starts on this rank's own column tiles (FC_GATHER_OVERLAP=0: gather, then pass 1)
  bool overlap_e = false;
  cudaStream_t ws3 = nullptr;
  cudaEvent_t e_fork{}, e_join{};
  CUtensorMap mE1l{}, mE2l{};             // the caller's slices (A rows and own column tiles)
  const void* map_l1 = nullptr;
  const void* map_l2 = nullptr;
  fc::StepResult* result_d = nullptr;   // device alias of result_h (mapped pinned memory)
  fc::StepResult* result_h = nullptr;   // written by the reduce kernel over PCIe: no D2H copy node
  cudaEvent_t done{}, fork{}, side_fork{}, side_join{};
  cudaStream_t ws = nullptr;     // context stream (capturable), joined to the caller's stream
  cudaStream_t ws2 = nullptr;    // side branch: reductions / tau updates off the critical path
  double* scal = nullptr;        // device {gamma_t, eps_t}
  bool use_graph = true;
  bool shared_q = true;          // K == 1: one Q pass, Q^T read by the dE2 GEMM
  bool prof = false;               // FC_PROFILE builds with FC_PROF=1: stamps into dbg_buf (fc_debug_counters)
  bool q_factor = true;          // FC_Q_FACTOR=0 forces the two-exponential Q path (A/B checks)
  bool fused_p1 = false;         // K == 1: row + column statistics from one S pass (FC_FUSED_P1=0: two passes)
  bool pdl = true;               // programmatic dependent launch between the step's kernels (FC_PDL=0: off)
  bool split_tail = false;       // similarity kernels: leftover tiles as half tiles (FC_SPLIT_TAIL=1; measured neutral)
  int gemm_drain = 0;            // FC_GEMM_DRAIN: stream-K unit-boundary cost in k-blocks (0: KB / 10)
  long long* dbg_buf = nullptr;   // profiling stamps: [launch 0: pass 1, 1: pass 2][pair][8], GEMM, anchor, prep, gathers
  struct GraphEntry {
    const void* key[6];
    cudaGraphExec_t exec;
    cudaGraph_t graph;                 // kept: its prep node addresses the per-step parameter update
    cudaGraphNode_t prep_node;
    cudaKernelNodeParams prep_params;  // captured launch shape of fc_prep_kernel
    const void* prep_e1;
    const void* prep_e2;
    fc::StepArgs prep_args;
    struct PeerNode {
      cudaGraphNode_t node;
      cudaKernelNodeParams kp;
      fc::PeerGather pg;
    };
    std::vector<PeerNode> peer_nodes;   // gathers whose sequence number changes every replay
  };
  std::vector<GraphEntry> graphs;
  // optional per-phase CUDA events (bench roofline): phases of the last step
  static constexpr int kPhases = 6;
  static constexpr int kAnchorBlock = 128;   // fc_anchor_kernel: 8 anchors (16-lane groups) per block
  static constexpr int kWeightsBlock = 64;   // fc_weights_kernel: thread per anchor, >= 80 blocks at B = 5120   // gatherE, prep, pass1, scalars, pass2, gemm
  bool timing = false;
  int ev_slots = 0, ev_cur = 0;        // ring of per-step event sets (no host sync between steps)
  std::vector<cudaEvent_t> ev;        // [ev_slots][kPhases + 1]
  bool debug_sync = false;
  void mark(int i, cudaStream_t st) {
    if (debug_sync) {
      cudaError_t e = cudaStreamSynchronize(st);
      std::fprintf(stderr, "[fc] phase %d reached (%s)\n", i, cudaGetErrorString(e));
    }
    if (timing) FC_CUDA(cudaEventRecord(ev[ev_cur * (kPhases + 1) + i], st));
  }
  // cached descriptors
  const void* map_e1 = nullptr;
  const void* map_e2 = nullptr;
  const void* map_o1 = nullptr;
  const void* map_o2 = nullptr;
  CUtensorMap mO[2];
  CUtensorMap mE1k, mE2k, mE1n, mE2n, mQ[2], mQt, mQo[2];
  fc::StepArgs args{};

  double* F(int i) const { return f64 + static_cast<size_t>(i) * Bl; }

  void init(const fc_config* c) {
    cfg = *c;
    K = cfg.world;
    rank = cfg.rank;
    Bl = cfg.local_batch;
    B = Bl * K;
    d = cfg.dim;
    if (K < 1 || rank < 0 || rank >= K) throw FcError{FC_ERR_CONFIG, "world/rank out of range"};
    if (Bl < 1) throw FcError{FC_ERR_CONFIG, "local_batch must be >= 1"};
    if (B < 2) throw FcError{FC_ERR_DEGENERATE_BATCH, "global batch must have >= 2 pairs"};
    if (d < 8 || d % 8 != 0) throw FcError{FC_ERR_UNSUPPORTED, "dim must be a positive multiple of 8"};
    if (cfg.n_train < B) throw FcError{FC_ERR_CONFIG, "n_train smaller than one global batch"};
    if (cfg.n_train > 0x7fffffffLL) throw FcError{FC_ERR_CONFIG, "n_train must fit int32 ids"};
    if (cfg.variant < 0 || cfg.variant > 6) throw FcError{FC_ERR_CONFIG, "unknown variant"};
    if (!(cfg.tau0 > 0.0) || cfg.tau_init < cfg.tau0) throw FcError{FC_ERR_CONFIG, "temperature.init/tau0"};
    indiv = is_individual(cfg.variant);
    track_u = cfg.variant != FC_OPENCLIP_MBCL;
    ldq = (B + 63) / 64 * 64;
    n_jt = (B + fc::kPairN - 1) / fc::kPairN;
    FC_CUDA(cudaSetDevice(cfg.device));
    n_sm = sm_count(cfg.device);
    my_dev = cfg.device;

    const size_t N = static_cast<size_t>(cfg.n_train);
    u1 = dalloc<double>(N);
    u2 = dalloc<double>(N);
    FC_CUDA(cudaMemset(u1, 0, N * 8));
    FC_CUDA(cudaMemset(u2, 0, N * 8));
    if (indiv) {
      tau1 = dalloc<double>(N); tau2 = dalloc<double>(N);
      m1 = dalloc<double>(N); v1 = dalloc<double>(N); m2 = dalloc<double>(N); v2 = dalloc<double>(N);
      s1 = dalloc<long long>(N); s2 = dalloc<long long>(N);
      std::vector<double> init(N, cfg.tau_init);
      FC_CUDA(cudaMemcpy(tau1, init.data(), N * 8, cudaMemcpyHostToDevice));
      FC_CUDA(cudaMemcpy(tau2, init.data(), N * 8, cudaMemcpyHostToDevice));
      for (double* p : {m1, v1, m2, v2}) FC_CUDA(cudaMemset(p, 0, N * 8));
      FC_CUDA(cudaMemset(s1, 0, N * 8));
      FC_CUDA(cudaMemset(s2, 0, N * 8));
    }
    tau_state = dalloc<fc::TauState>(1);
    fc::TauState ts{cfg.tau_init, 0.0, 0.0, 0, 0, 0};
    FC_CUDA(cudaMemcpy(tau_state, &ts, sizeof(ts), cudaMemcpyHostToDevice));

    if (K > 1) {
      e1g = dalloc<__nv_bfloat16>(2 * static_cast<size_t>(B) * d);
      e2g = dalloc<__nv_bfloat16>(2 * static_cast<size_t>(B) * d);
      ncclUniqueId id;
      std::memcpy(&id, cfg.nccl_id, sizeof(id));
      FC_NCCL(ncclCommInitRank(&comm, K, id, rank));
      check_collective_shape();
    }
    diag = dalloc<float>(B);
    rowstat = dalloc<float2>(2 * static_cast<size_t>(Bl));
    partial = dalloc<float2>(2 * static_cast<size_t>(Bl) * n_jt * 4);
    if (K == 1)   // [ceil(B/32)][n_slots = 2 per pair row block][32]: 256-byte warp stores
      col_partial = dalloc<float2>(static_cast<size_t>((Bl + fc::kPairM - 1) / fc::kPairM) * 2 * ((B + 31) / 32 * 32));
    clamps = dalloc<unsigned long long>(1);
    bounds = dalloc<float>(2 * 4 * fc::kMaxPeers);   // one {norm1, norm2, kappa, -} slot per rank and parity
    FC_CUDA(cudaMemset(bounds, 0, 2 * 4 * fc::kMaxPeers * sizeof(float)));
    f64 = dalloc<double>(static_cast<size_t>(Bl) * 13);   // F(0) .. F(12) below
    nblk = (Bl * fc::kAnchorLanes + kAnchorBlock - 1) / kAnchorBlock;
    pstride = (7 * Bl + 3 * nblk + 1) & ~1;   // even: 16-byte slices for the peer gather
    send = dalloc<double>(static_cast<size_t>(pstride));
    recv = K > 1 ? dalloc<double>(static_cast<size_t>(K) * pstride) : send;
    red = dalloc<double>(2);
    par = dalloc<float>(8 * static_cast<size_t>(n_jt) * fc::kPairN);
    FC_CUDA(cudaMemset(par, 0, 8 * static_cast<size_t>(n_jt) * fc::kPairN * 4));
    rcoef = dalloc<float>(Bl);
    q = dalloc<__nv_bfloat16>(2 * static_cast<size_t>(Bl) * ldq);
    err = dalloc<int>(1);
    idset_slots = 64;
    while (idset_slots < 2 * Bl) idset_slots *= 2;
    idset = dalloc<unsigned long long>(idset_slots);
    FC_CUDA(cudaMemset(idset, 0, idset_slots * sizeof(unsigned long long)));
    step_tag = dalloc<unsigned long long>(1);
    FC_CUDA(cudaMemset(step_tag, 0, sizeof(unsigned long long)));
    rs = K > 1 && cfg.reduction == 1;
    if (cfg.reduction < 0 || cfg.reduction > 1) throw FcError{FC_ERR_CONFIG, "fabric.reduction: expected 0 (fastclip) or 1 (openclip_rs)"};
    if (rs) {
      if (Bl % 64 != 0) throw FcError{FC_ERR_UNSUPPORTED, "openclip_rs needs a local batch that is a multiple of 64"};
      rs_part = dalloc<float>(2 * static_cast<size_t>(B) * d);
      rs_shard = dalloc<float>(2 * static_cast<size_t>(Bl) * d);
      for (int s2 = 0; s2 < 2; ++s2) {
        // Q'_C^T / Q'_R^T as MN-major A operands (64 x 64 atoms of the row-major [Bl][ldq] Q')
        mQtRS[s2] = make_map(q + static_cast<size_t>(1 - s2) * Bl * ldq, ldq, Bl, static_cast<uint64_t>(ldq) * 2, 64, 64);
        mPart[s2] = make_map(rs_part + static_cast<size_t>(s2) * B * d, d, B, static_cast<uint64_t>(d) * 4, 32, 32,
                             CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
      }
    }
    if (K > 1) setup_peers();
    FC_CUDA(cudaMemset(err, 0, sizeof(int)));
    FC_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&result_h), sizeof(fc::StepResult), cudaHostAllocMapped));
    std::memset(result_h, 0, sizeof(*result_h));
    FC_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&result_d), result_h, 0));
    FC_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    FC_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    FC_CUDA(cudaStreamCreateWithFlags(&ws, cudaStreamNonBlocking));
    {
      int lo = 0, hi = 0;   // numerically greatest = lowest priority
      FC_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      FC_CUDA(cudaStreamCreateWithPriority(&ws2, cudaStreamNonBlocking, lo));
    }
    FC_CUDA(cudaEventCreateWithFlags(&side_fork, cudaEventDisableTiming));
    FC_CUDA(cudaEventCreateWithFlags(&side_join, cudaEventDisableTiming));
    scal = dalloc<double>(2);
    if (const char* e = std::getenv("FC_GRAPH")) use_graph = atoi(e) != 0;
    shared_q = K == 1;
    if (const char* e = std::getenv("FC_DEBUG_SYNC")) debug_sync = atoi(e) != 0;
#ifdef FC_PROFILE
    if (const char* e = std::getenv("FC_PROF")) prof = atoi(e) != 0;
#endif
    if (const char* e = std::getenv("FC_Q_FACTOR")) q_factor = atoi(e) != 0;
    fused_p1 = K == 1;
    if (const char* e = std::getenv("FC_PDL")) pdl = atoi(e) != 0;
    if (const char* e = std::getenv("FC_SPLIT_TAIL")) split_tail = atoi(e) != 0;
    if (const char* e = std::getenv("FC_GEMM_DRAIN")) gemm_drain = atoi(e);
    if (const char* e = std::getenv("FC_FUSED_P1")) fused_p1 = fused_p1 && atoi(e) != 0;
    if (prof) dbg_buf = dalloc<long long>(2 * 2688 + 160 * 16 + 8192);
    if (dbg_buf && use_peer) {   // gather stamps after the anchor / prep stamps
      for (int q2 = 0; q2 < 2; ++q2) {
        pg_e[q2].dbg = dbg_buf + 2 * 2688 + 160 * 16 + 6000;
        pg_p[q2].dbg = pg_e[q2].dbg + 4;
      }
    }
    if (debug_sync) use_graph = false;
    if (const char* e = std::getenv("FC_SHARED_Q")) shared_q = shared_q && atoi(e) != 0;
    if (const char* e = std::getenv("FC_DUP_CHECK")) dup_check = atoi(e) != 0;
    if (const char* e = std::getenv("FC_PEER_BULK")) peer_bulk = atoi(e) != 0;
    if (use_peer) {
      overlap_e = !peer_bulk;
      if (const char* e = std::getenv("FC_GATHER_OVERLAP")) overlap_e = overlap_e && atoi(e) != 0;
      // pass 1 waits inside its grid for the gather's flags: a gather CTA must fit beside a pass-1
      // CTA on the same SM (registers, shared memory, threads), else the overlap could deadlock
      if (overlap_e) overlap_e = gather_fits_beside_passes();
      if (overlap_e) {
        int lo = 0, hi = 0;
        FC_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        FC_CUDA(cudaStreamCreateWithPriority(&ws3, cudaStreamNonBlocking, hi));
        FC_CUDA(cudaEventCreateWithFlags(&e_fork, cudaEventDisableTiming));
        FC_CUDA(cudaEventCreateWithFlags(&e_join, cudaEventDisableTiming));
      }
    }
    if (const char* e = std::getenv("FC_TEST_DELAY_US")) test_delay_ns = K > 1 ? atoll(e) * 1000LL : 0;
    FC_CUDA(fc::sim_set_smem());
    FC_CUDA(fc::gemm_set_smem());
    // side-branch kernels run beside persistent similarity CTAs: ask for the max-shared
    // carveout so the SM configuration they land on never has to change for a pass-2 CTA
    FC_CUDA(cudaFuncSetAttribute(fc::fc_reduce_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 cudaSharedmemCarveoutMaxShared));
    // prep and the per-anchor kernel run while the next similarity pass's CTAs (227 KB of
    // shared memory each) take their SMs (programmatic launch)
    FC_CUDA(cudaFuncSetAttribute(fc::fc_prep_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 cudaSharedmemCarveoutMaxShared));
    FC_CUDA(cudaFuncSetAttribute(fc::fc_anchor_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 cudaSharedmemCarveoutMaxShared));
    for (bool lean : {false, true})
      FC_CUDA(cudaFuncSetAttribute(fc::peer_gather_kernel_fn(lean), cudaFuncAttributePreferredSharedMemoryCarveout,
                                   cudaSharedmemCarveoutMaxShared));
    FC_CUDA(cudaFuncSetAttribute(fc::fc_indiv_update_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 cudaSharedmemCarveoutMaxShared));
    mQ[0] = make_map(q, ldq, Bl, static_cast<uint64_t>(ldq) * 2, 64, 128);
    mQ[1] = make_map(q + static_cast<size_t>(Bl) * ldq, ldq, Bl, static_cast<uint64_t>(ldq) * 2, 64, 128);
    mQt = make_map(q, ldq, Bl, static_cast<uint64_t>(ldq) * 2, 64, 64);   // Q^T as MN-major A (K = 1)
    for (int s2 = 0; s2 < 2; ++s2)   // Q-pass tile stores: 32 rows x 32 bf16, 64-byte swizzle
      mQo[s2] = make_map(q + static_cast<size_t>(s2) * Bl * ldq, ldq, Bl, static_cast<uint64_t>(ldq) * 2, 32, 32,
                         CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, CU_TENSOR_MAP_SWIZZLE_64B);
    build_args();
  }

  void build_args() {
    fc::StepArgs& a = args;
    a.B = B; a.Bl = Bl; a.d = d; a.world = K; a.rank = rank; a.row0 = rank * Bl; a.n_jt = n_jt;
    a.variant = cfg.variant; a.individual = indiv; a.track_u = track_u; a.scale_by_tau = cfg.scale_by_tau;
    a.lr_decay_enabled = cfg.lr_decay_enabled;
    a.n_train = cfg.n_train;
    a.rho = cfg.rho; a.tau_lr = cfg.tau_lr; a.tau0 = cfg.tau0; a.beta1 = cfg.beta1; a.beta2 = cfg.beta2;
    a.adam_eps = cfg.adam_eps; a.lr_decay_threshold = cfg.lr_decay_threshold; a.lr_decay_factor = cfg.lr_decay_factor;
    a.diag = diag;
    a.u1_tab = u1; a.u2_tab = u2; a.tau1_tab = tau1; a.tau2_tab = tau2;
    a.m1_tab = m1; a.v1_tab = v1; a.s1_tab = s1; a.m2_tab = m2; a.v2_tab = v2; a.s2_tab = s2;
    a.tau_state = tau_state;
    a.rowstat_R = rowstat; a.rowstat_C = rowstat + Bl;
    a.partial_R = partial; a.partial_C = partial + static_cast<size_t>(Bl) * n_jt * 4;
    a.clamps = clamps;
    a.bounds = bounds + 4 * rank;
    a.t_loc1 = F(0); a.t_loc2 = F(1);
    a.sum1 = F(2); a.dx1 = F(3); a.sum2 = F(4); a.dx2 = F(5);
    a.g1 = F(6); a.g2 = F(7); a.u1 = F(8); a.u2 = F(9);
    a.term_a = F(10); a.term_b = F(11); a.term_loss = F(12);
    a.gt1 = send + 5 * static_cast<size_t>(Bl); a.gt2 = send + 6 * static_cast<size_t>(Bl);   // payload columns
    a.send = send; a.recv = recv;
    a.pstride = pstride; a.nblk = nblk;
    const size_t np = static_cast<size_t>(n_jt) * fc::kPairN;
    a.kap1 = par; a.bet1 = par + np; a.coef1 = par + 2 * np;
    a.kap2 = par + 3 * np; a.bet2 = par + 4 * np; a.coef2 = par + 5 * np;
    a.fac1 = par + 6 * np; a.fac2 = par + 7 * np;
    a.rcoef = rcoef;
    a.blockpart = send + 7 * static_cast<size_t>(Bl);
    a.red = red; a.err = err; a.result = result_d;
    a.step_tag = step_tag;
  }

  // Every rank must run the same step shape (variant, batch, dim, table size, world): the
  // reference's rendezvous throws CollectiveShapeError when peers disagree on an op's shape
  // (fabric.cpp:130-138); here the ranks compare their configurations once, at creation.
  void check_collective_shape() {
    const long long mine[6] = {cfg.variant, Bl, d, cfg.n_train, K, cfg.scale_by_tau};
    cudaStream_t s0;
    FC_CUDA(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
    long long* dv = dalloc<long long>(6 * (K + 1));
    FC_CUDA(cudaMemcpy(dv + 6 * K, mine, sizeof(mine), cudaMemcpyHostToDevice));
    FC_NCCL(ncclAllGather(dv + 6 * K, dv, 6, ncclInt64, comm, s0));
    FC_CUDA(cudaStreamSynchronize(s0));
    std::vector<long long> all(6 * static_cast<size_t>(K));
    FC_CUDA(cudaMemcpy(all.data(), dv, all.size() * sizeof(long long), cudaMemcpyDeviceToHost));
    cudaFree(dv);
    cudaStreamDestroy(s0);
    for (int k = 0; k < K; ++k)
      for (int f = 0; f < 6; ++f)
        if (all[6 * k + f] != mine[f])
          throw FcError{FC_ERR_COLLECTIVE_SHAPE, "rank " + std::to_string(k) + " runs a different step shape "
                                                 "(variant / local batch / dim / n_train / world / scale_by_tau)"};
  }

  // CUDA IPC mappings of every rank's gather destinations and flag arrays; handles travel
  // over the NCCL communicator once. Falls back to NCCL gathers when a pair of GPUs cannot
  // map each other's memory.
  void setup_peers() {
    if (const char* e = std::getenv("FC_PEER"))
      if (atoi(e) == 0) return;
    if (K > fc::kMaxPeers || Bl % 4 != 0) return;   // 16-byte parameter slices
    // the ranks' device ordinals (one node), then every pair must be able to map the other
    cudaStream_t s0;
    FC_CUDA(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
    int* ddev = dalloc<int>(K + 1);
    FC_CUDA(cudaMemcpy(ddev + K, &my_dev, sizeof(int), cudaMemcpyHostToDevice));
    FC_NCCL(ncclAllGather(ddev + K, ddev, 1, ncclInt32, comm, s0));
    FC_CUDA(cudaStreamSynchronize(s0));
    std::vector<int> devs(K);
    FC_CUDA(cudaMemcpy(devs.data(), ddev, K * sizeof(int), cudaMemcpyDeviceToHost));
    cudaFree(ddev);
    int ok = 1;
    for (int k = 0; k < K; ++k) {
      if (devs[k] == my_dev) continue;
      int can = 0;
      if (cudaDeviceCanAccessPeer(&can, my_dev, devs[k]) != cudaSuccess || !can) ok = 0;
    }
    // every rank must agree: all-reduce the capability (min) over the communicator
    int* dok = dalloc<int>(1);
    FC_CUDA(cudaMemcpy(dok, &ok, sizeof(int), cudaMemcpyHostToDevice));
    FC_NCCL(ncclAllReduce(dok, dok, 1, ncclInt32, ncclMin, comm, s0));
    FC_CUDA(cudaStreamSynchronize(s0));
    FC_CUDA(cudaMemcpy(&ok, dok, sizeof(int), cudaMemcpyDeviceToHost));
    cudaFree(dok);
    if (!ok) {
      cudaStreamDestroy(s0);
      return;
    }
    pflags = dalloc<unsigned long long>(2 * fc::kMaxPeers + 1);
    FC_CUDA(cudaMemset(pflags, 0, (2 * fc::kMaxPeers + 1) * sizeof(unsigned long long)));
    ptickets = dalloc<unsigned>(2);
    FC_CUDA(cudaMemset(ptickets, 0, 2 * sizeof(unsigned)));
    void* mine[6] = {e1g, e2g, recv, pflags, par, bounds};
    cudaIpcMemHandle_t h[6];
    for (int i = 0; i < 6; ++i) FC_CUDA(cudaIpcGetMemHandle(&h[i], mine[i]));
    uint8_t* dh = dalloc<uint8_t>(sizeof(h) * (K + 1));
    FC_CUDA(cudaMemcpy(dh + sizeof(h) * K, h, sizeof(h), cudaMemcpyHostToDevice));
    FC_NCCL(ncclAllGather(dh + sizeof(h) * K, dh, sizeof(h), ncclUint8, comm, s0));
    FC_CUDA(cudaStreamSynchronize(s0));
    cudaStreamDestroy(s0);
    std::vector<cudaIpcMemHandle_t> all(6 * static_cast<size_t>(K));
    FC_CUDA(cudaMemcpy(all.data(), dh, sizeof(h) * K, cudaMemcpyDeviceToHost));
    cudaFree(dh);
    void* peer[6][fc::kMaxPeers] = {};
    for (int k = 0; k < K; ++k)
      for (int i = 0; i < 6; ++i) {
        if (k == rank) {
          peer[i][k] = mine[i];
        } else {
          FC_CUDA(cudaIpcOpenMemHandle(&peer[i][k], all[6 * k + i], cudaIpcMemLazyEnablePeerAccess));
          peer_maps.push_back(peer[i][k]);
        }
      }
    // E gather: the two embedding slices. Payload gather: [u|t|id|gt|partials] plus this
    // rank's slice of the 8 pass-2 parameter arrays (kappa, beta, coef, fac x 2 tracks), so the
    // pass-2 parameters of every anchor arrive ready-made (no weights kernel on the step path)
    const size_t np = static_cast<size_t>(n_jt) * fc::kPairN;
    const char* tmo = std::getenv("FC_PEER_TIMEOUT_MS");   // a peer that stops stepping: poison after this long
    const long long timeout_ns = (tmo ? atoll(tmo) : 60000LL) * 1000000LL;
    const size_t ebytes = static_cast<size_t>(B) * d * 2;   // one parity's gathered rows
    for (int q2 = 0; q2 < 2; ++q2) {
      fc::PeerGather& ge = pg_e[q2];
      fc::PeerGather& gpl = pg_p[q2];
      const float* bslot = bounds + q2 * 4 * fc::kMaxPeers + 4 * rank;
      ge = fc::PeerGather{};
      ge.bytes[0] = ge.bytes[1] = static_cast<size_t>(Bl) * d * 2;
      ge.bytes[2] = 16;   // this rank's bounds slot (norm maxima written by prep)
      ge.src[2] = reinterpret_cast<const uint8_t*>(bslot);
      ge.n_src = 3;
      gpl = fc::PeerGather{};
      gpl.bytes[0] = static_cast<size_t>(pstride) * 8;
      gpl.src[0] = reinterpret_cast<const uint8_t*>(send);
      gpl.n_src = 1 + 8 + 1;
      for (int j = 0; j < 8; ++j) {
        gpl.bytes[1 + j] = static_cast<size_t>(Bl) * 4;
        gpl.src[1 + j] = reinterpret_cast<const uint8_t*>(par + j * np + static_cast<size_t>(rank) * Bl);
      }
      gpl.bytes[9] = 16;   // bounds slot again, now with the kappa maximum of the anchor kernel
      gpl.src[9] = reinterpret_cast<const uint8_t*>(bslot);
      for (fc::PeerGather* g : {&ge, &gpl}) {
        g->world = K;
        g->rank = rank;
        g->err = err;
        g->timeout_ns = timeout_ns;
        g->my_abort = pflags + 2 * fc::kMaxPeers;
      }
      for (int k = 0; k < K; ++k) {
        ge.dst[0][k] = static_cast<uint8_t*>(peer[0][k]) + q2 * ebytes;
        ge.dst[1][k] = static_cast<uint8_t*>(peer[1][k]) + q2 * ebytes;
        gpl.dst[0][k] = static_cast<uint8_t*>(peer[2][k]);
        for (int j = 0; j < 8; ++j)
          gpl.dst[1 + j][k] = static_cast<uint8_t*>(peer[4][k]) + j * np * 4;
        uint8_t* pb = static_cast<uint8_t*>(peer[5][k]) + q2 * 4 * fc::kMaxPeers * sizeof(float);
        ge.dst[2][k] = pb;   // norm maxima slot
        gpl.dst[9][k] = pb;
        ge.peer_flag[k] = static_cast<unsigned long long*>(peer[3][k]);
        gpl.peer_flag[k] = static_cast<unsigned long long*>(peer[3][k]) + fc::kMaxPeers;
        ge.peer_abort[k] = gpl.peer_abort[k] = static_cast<unsigned long long*>(peer[3][k]) + 2 * fc::kMaxPeers;
      }
      ge.my_flag = pflags;
      gpl.my_flag = pflags + fc::kMaxPeers;
      ge.ticket = ptickets;
      gpl.ticket = ptickets + 1;
    }
    use_peer = true;
  }

  // One (lean) gather CTA of kGatherThreads beside one pass-1 / pass-2 CTA on an SM: shared memory (+ the
  // per-CTA reservation), threads, and registers per SM sub-partition -- warps are dealt
  // round-robin over the four sub-partitions, each with a quarter of the register file, so the
  // pass-1 CTA's 18 warps leave its two fuller sub-partitions the least room; every alignment of
  // the gather CTA's warps against them must fit.
  static constexpr int kGatherThreads = 128;
  bool gather_fits_beside_passes() const {
    for (int mode : {fc::kSimStats, fc::kSimQ})
      if (!gather_fits_beside(mode)) return false;
    return true;
  }
  bool gather_fits_beside(int mode) const {
    cudaFuncAttributes fs{}, fg{};
    if (fc::sim_attributes(mode, &fs) != cudaSuccess ||
        cudaFuncGetAttributes(&fg, fc::peer_gather_kernel_fn(true)) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    int smem_sm = 0, regs_sm = 0, thr_sm = 0, resv = 0;
    cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, my_dev);
    cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, my_dev);
    cudaDeviceGetAttribute(&thr_sm, cudaDevAttrMaxThreadsPerMultiProcessor, my_dev);
    cudaDeviceGetAttribute(&resv, cudaDevAttrReservedSharedMemoryPerBlock, my_dev);
    auto warp_regs = [](int per_thread) { return (per_thread * 32 + 255) / 256 * 256; };
    const int sim_warps = fc::kSimThreads / 32, g_warps = kGatherThreads / 32;
    bool regs_ok = true;
    for (int rot = 0; rot < 4; ++rot)
      for (int sp = 0; sp < 4; ++sp) {
        const int ws_ = (sim_warps - sp + 3) / 4;                    // pass-1 warps on sub-partition sp
        const int wg = (g_warps - ((sp - rot + 4) % 4) + 3) / 4;     // gather warps there (rotated start)
        regs_ok = regs_ok && ws_ * warp_regs(fs.numRegs) + wg * warp_regs(fg.numRegs) <= regs_sm / 4;
      }
    const long smem = static_cast<long>(fc::kSimSmemBytes) + fs.sharedSizeBytes + resv + fg.sharedSizeBytes + resv;
    return regs_ok && smem <= smem_sm && fc::kSimThreads + kGatherThreads <= thr_sm;
  }

  void ensure_maps(const void* e1, const void* e2) {
    if (e1 == map_e1 && e2 == map_e2) return;
    const uint64_t rb = static_cast<uint64_t>(d) * 2;
    mE1k = make_map(e1, d, B, rb, 64, 128);
    mE2k = make_map(e2, d, B, rb, 64, 128);
    mE1n = make_map(e1, d, B, rb, 64, 64);
    mE2n = make_map(e2, d, B, rb, 64, 64);
    map_e1 = e1;
    map_e2 = e2;
  }

  void balance_units(fc::GemmParams& gp, int n_clusters) const { balance_stream_k(gp, n_clusters, gemm_drain); }

  int pair_grid(long items) const {
    long pairs = std::min<long>(n_sm / 2, items);
    return static_cast<int>(std::max<long>(1, pairs) * 2);
  }

  // Validates, stages the step scalars and runs the step on the context stream: replayed
  // from a CUDA graph captured per (input, output) pointer set, or enqueued directly.
  void step(const fc_step_in* in, fc_step_out* out, cudaStream_t caller) {
    nvtx3::scoped_range nvtx_step{"fc_loss_step"};
    if (!in || !out || !in->e1 || !in->e2 || !in->ids || !out->de1 || !out->de2)
      throw FcError{FC_ERR_SHAPE, "fc_loss_step: null input/output pointer"};
    if (in->eps < 0.0) throw FcError{FC_ERR_DOMAIN, "epsilon must be non-negative"};
    if (track_u && (!(in->gamma > 0.0) || in->gamma > 1.0)) throw FcError{FC_ERR_DOMAIN, "gamma must be in (0,1]"};
    ++seq;   // every rank calls step() the same number of times: the peer-gather handshake value
    if (use_graph && !timing) {   // phase timing: direct launches (events between kernels)
      // one graph per (input, output) pointer set and step parity (the gather buffers alternate)
      const void* key[6] = {in->e1, in->e2, in->ids, out->de1, out->de2,
                            reinterpret_cast<const void*>(static_cast<uintptr_t>(parity()))};
      GraphEntry* ge = nullptr;
      for (auto& g : graphs)
        if (std::memcmp(g.key, key, sizeof(key)) == 0) ge = &g;
      if (!ge) {
        if (graphs.size() >= 8) {
          cudaGraphExecDestroy(graphs.front().exec);
          cudaGraphDestroy(graphs.front().graph);
          graphs.erase(graphs.begin());
        }
        GraphEntry g{};
        nvtx3::scoped_range nvtx_cap{"fc_loss_step: capture + instantiate the step graph"};
        FC_CUDA(cudaStreamBeginCapture(ws, cudaStreamCaptureModeThreadLocal));
        try {
          enqueue(in, out, ws);
        } catch (...) {
          cudaStreamEndCapture(ws, &g.graph);
          if (g.graph) cudaGraphDestroy(g.graph);
          throw;
        }
        FC_CUDA(cudaStreamEndCapture(ws, &g.graph));
        FC_CUDA(cudaGraphInstantiate(&g.exec, g.graph, 0));
        // the prep kernel node carries the step scalars (gamma_t, eps_t) as parameters
        size_t n = 0;
        FC_CUDA(cudaGraphGetNodes(g.graph, nullptr, &n));
        std::vector<cudaGraphNode_t> nodes(n);
        FC_CUDA(cudaGraphGetNodes(g.graph, nodes.data(), &n));
        for (auto nd : nodes) {
          cudaGraphNodeType t;
          FC_CUDA(cudaGraphNodeGetType(nd, &t));
          if (t != cudaGraphNodeTypeKernel) continue;
          cudaKernelNodeParams kp{};
          if (cudaGraphKernelNodeGetParams(nd, &kp) != cudaSuccess) {   // e.g. NCCL's own kernels
            cudaGetLastError();
            continue;
          }
          if (kp.func == reinterpret_cast<void*>(fc::fc_prep_kernel)) {
            g.prep_node = nd;
            g.prep_params = kp;
          }
          if (kp.func == fc::peer_gather_kernel_fn(false) || kp.func == fc::peer_gather_kernel_fn(true)) {
            GraphEntry::PeerNode pn{nd, kp, *static_cast<fc::PeerGather*>(kp.kernelParams[0])};
            g.peer_nodes.push_back(pn);
          }
        }
        if (!g.prep_node) throw FcError{FC_ERR_CUDA, "captured step graph has no prep node"};
        g.prep_e1 = last_prep_e1;
        g.prep_e2 = last_prep_e2;
        g.prep_args = last_prep_args;
        std::memcpy(g.key, key, sizeof(key));
        graphs.push_back(g);
        ge = &graphs.back();
      }
      double gamma = in->gamma, eps = in->eps;
      const void* e1 = ge->prep_e1;
      const void* e2 = ge->prep_e2;
      unsigned long long sq = seq;
      void* args[6] = {&e1, &e2, &ge->prep_args, &gamma, &eps, &sq};
      cudaKernelNodeParams kp = ge->prep_params;
      kp.kernelParams = args;
      kp.extra = nullptr;
      FC_CUDA(cudaGraphExecKernelNodeSetParams(ge->exec, ge->prep_node, &kp));
      for (auto& pn : ge->peer_nodes) {
        pn.pg.seq = seq;
        void* pargs[1] = {&pn.pg};
        cudaKernelNodeParams pk = pn.kp;
        pk.kernelParams = pargs;
        pk.extra = nullptr;
        FC_CUDA(cudaGraphExecKernelNodeSetParams(ge->exec, pn.node, &pk));
      }
      FC_CUDA(cudaGraphLaunch(ge->exec, caller));   // the replay joins the caller's stream directly
      FC_CUDA(cudaEventRecord(done, caller));        // fc_step_scalars_get waits on it
    } else {
      FC_CUDA(cudaEventRecord(fork, caller));
      FC_CUDA(cudaStreamWaitEvent(ws, fork, 0));
      enqueue(in, out, ws);
      FC_CUDA(cudaEventRecord(done, ws));
      FC_CUDA(cudaStreamWaitEvent(caller, done, 0));
    }
    if (timing) ev_last = ev_cur, ev_cur = (ev_cur + 1) % ev_slots;
    book_step();
  }
  int ev_last = 0;
  const void* last_prep_e1 = nullptr;   // arguments of the last enqueued prep kernel (graph capture)
  const void* last_prep_e2 = nullptr;
  fc::StepArgs last_prep_args{};

  int parity() const { return K > 1 ? static_cast<int>(seq & 1) : 0; }

  void enqueue(const fc_step_in* in, fc_step_out* out, cudaStream_t st) {
    const __nv_bfloat16* E1 = static_cast<const __nv_bfloat16*>(in->e1);
    const __nv_bfloat16* E2 = static_cast<const __nv_bfloat16*>(in->e2);
    mark(0, st);
    fc::StepArgs a = args;
    const int par = parity();
    float* bnd = bounds + par * 4 * fc::kMaxPeers;   // this step's bounds slots (one per rank)
    a.bounds = bnd + 4 * rank;
    a.ids = in->ids;
    a.gscale = static_cast<float>(1.0 / (static_cast<double>(Bl) * static_cast<double>(B - 1)));
    a.scal = scal;
    if (prof) a.dbg = dbg_buf + 2 * 2688 + 160 * 16;
    // prep: with peer memory every rank preps only its own anchors, BEFORE the gather (the
    // diagonal and tau^t of non-local anchors are never needed: their pass-2 parameters arrive
    // ready-made); its norm maxima sit in this rank's bounds slot, which the gather copies
    // into every rank (consumers take the max over the slots). Otherwise prep covers G after
    // the gather.
    const bool local_prep = K > 1 && use_peer;
    auto launch_prep = [&](const __nv_bfloat16* p1, const __nv_bfloat16* p2, int row0_, int rows) {
      a.prep_row0 = row0_;
      a.prep_rows = rows;
      // bounds were zeroed by the previous step's GEMM (and at creation)
      fc::fc_prep_kernel<<<(rows * 32 + 127) / 128, 128, 0, st>>>(p1, p2, a, in->gamma, in->eps, seq);   // one wave
      FC_CUDA(cudaGetLastError());
      last_prep_e1 = p1;
      last_prep_e2 = p2;
      last_prep_args = a;
    };
    const __nv_bfloat16* E1l = E1;   // the caller's slices
    const __nv_bfloat16* E2l = E2;
    const bool overlap = K > 1 && overlap_e;
    // pass 2 beside the payload gather as well, except for the reduce-scatter strategy (its mask
    // kernel zeroes the gathered parameters of the other ranks' anchors before pass 2)
    const bool overlap2 = overlap && !rs;
    if (overlap) {
      // the embedding gather on its own stream from the step's start: pass 1 reads own column
      // tiles from the caller's slices and each rank's gathered rows after that rank's flag
      FC_CUDA(cudaEventRecord(e_fork, st));
      FC_CUDA(cudaStreamWaitEvent(ws3, e_fork, 0));
      fc::PeerGather g = pg_e[par];
      g.src[0] = reinterpret_cast<const uint8_t*>(E1);
      g.src[1] = reinterpret_cast<const uint8_t*>(E2);
      g.n_src = 2;   // no bounds slot: pass 1 checks the clamp per chunk, pass 2 gets the slots with the payload
      g.seq = seq;
      g.wait_src = -1;
      FC_CUDA(fc::launch_peer_gather(g, n_sm, kGatherThreads, ws3, false, true));
      FC_CUDA(cudaEventRecord(e_join, ws3));
      if (E1 != map_l1 || E2 != map_l2) {
        const uint64_t rbytes = static_cast<uint64_t>(d) * 2;
        mE1l = make_map(E1, d, Bl, rbytes, 64, 128);
        mE2l = make_map(E2, d, Bl, rbytes, 64, 128);
        map_l1 = E1;
        map_l2 = E2;
      }
    }
    if (local_prep) launch_prep(E1, E2, rank * Bl, Bl);
    if (K > 1) {
      if (overlap) {
        // launched above
      } else if (use_peer) {   // NVLink stores into every rank's e1g / e2g, flag handshake
        fc::PeerGather g = pg_e[par];
        g.src[0] = reinterpret_cast<const uint8_t*>(E1);
        g.src[1] = reinterpret_cast<const uint8_t*>(E2);
        g.seq = seq;
        // programmatic launch after the local prep: the E slices go out while prep runs; the
        // bounds slot (source 2, prep's norm maxima) is sent after griddepcontrol.wait. Pass 1
        // waits for this grid, which completes only after prep did.
        g.wait_src = 2;
        g.bulk = peer_bulk ? 1 : 0;
        FC_CUDA(fc::launch_peer_gather(g, n_sm, 256, st, pdl && !timing));
      } else {
        FC_NCCL(ncclGroupStart());
        FC_NCCL(ncclAllGather(E1, e1g + par * static_cast<size_t>(B) * d, static_cast<size_t>(Bl) * d * 2, ncclUint8,
                              comm, st));
        FC_NCCL(ncclAllGather(E2, e2g + par * static_cast<size_t>(B) * d, static_cast<size_t>(Bl) * d * 2, ncclUint8,
                              comm, st));
        FC_NCCL(ncclGroupEnd());
      }
      E1 = e1g + par * static_cast<size_t>(B) * d;
      E2 = e2g + par * static_cast<size_t>(B) * d;
    }
    ensure_maps(E1, E2);
    mark(1, st);
    if (!local_prep) launch_prep(E1, E2, 0, B);

    // ---- pass 1: row statistics of S[L,G] (segment R) and S^T[L,G] (segment C) ----
    fc::SimParams sp{};
    sp.nseg = 2;
    sp.d = d;
    sp.ldq = ldq;
    sp.n_jt = n_jt;
    for (int s = 0; s < 2; ++s) {
      fc::SimSeg& g = sp.seg[s];
      g.rows = Bl;
      g.a_row0 = rank * Bl;
      g.cols = B;
      g.row_stat = s ? a.rowstat_C : a.rowstat_R;
      g.partial = s ? a.partial_C : a.partial_R;
      sp.n_rb[s] = (Bl + fc::kPairM - 1) / fc::kPairM;
    }
    sp.n_items = (sp.n_rb[0] + sp.n_rb[1]) * n_jt;
    sp.clamps = clamps;
    sp.bounds = bnd;
    sp.n_bounds = K;
    sp.ids = in->ids;
    sp.n_ids = Bl;
    sp.idset = dup_check ? idset : nullptr;
    sp.idset_mask = idset_slots - 1;
    sp.step_tag = step_tag;
    sp.err = err;
    sp.zero0 = reinterpret_cast<float4*>(out->de1);   // the GEMM's reduce-add targets
    sp.zero1 = reinterpret_cast<float4*>(out->de2);
    sp.zero_n4 = static_cast<long long>(Bl) * d / 4;
    sp.split_tail = split_tail ? 1 : 0;
    if (prof) sp.dbg_out = dbg_buf;
    CUtensorMap mA[2] = {mE1k, mE2k}, mB[2] = {mE2k, mE1k};
    mark(2, st);
    if (overlap) {
      sp.local_first = 1;
      sp.col_lo = rank * Bl;
      sp.jt_lo = (rank * Bl + fc::kPairN - 1) / fc::kPairN;
      sp.n_loc = std::max(0, std::min((rank + 1) * Bl / fc::kPairN, n_jt) - sp.jt_lo);
      sp.rows_per_src = Bl;
      sp.src_flag = pg_e[par].my_flag;
      sp.abort_flag = pg_e[par].my_abort;
      sp.timeout_ns = pg_e[par].timeout_ns;
      sp.exact_bounds = 1;
      sp.n_bounds = 0;
      sp.split_tail = 0;

      CUtensorMap mAl[2] = {mE1l, mE2l}, mOwn[2] = {mE2l, mE1l};
      // at least two tiles per pair: the local-first split keeps every pair's remote share >= 0
      FC_CUDA(fc::launch_sim(fc::kSimStats, sp, mAl, mB, mOwn, pair_grid(sp.n_items / 2), st, nullptr, pdl && !timing));
      sp.local_first = 0;
      sp.exact_bounds = 0;
      sp.n_bounds = K;
      sp.split_tail = split_tail ? 1 : 0;
    } else
    if (fused_p1) {
      // K = 1: segment C is S^T -- its row statistics are the column statistics of the
      // segment-R tiles, collected in the same epilogue (S is multiplied once)
      sp.nseg = 1;
      sp.n_rb[1] = 0;
      sp.n_items = sp.n_rb[0] * n_jt;
      sp.seg[0].col_stat = a.rowstat_C;
      sp.col_partial = col_partial;
      sp.n_slots = sp.n_rb[0] * 2;   // one column partial per CTA of each pair row block
      sp.fuse_fast = indiv ? 0 : 1;
      a.col_partial = col_partial;
      a.col_slots = sp.n_slots;
      FC_CUDA(fc::launch_sim(fc::kSimFused, sp, mA, mB, nullptr, pair_grid(sp.n_items), st, nullptr, pdl && !timing));
    } else {
      a.col_slots = 0;
      FC_CUDA(fc::launch_sim(fc::kSimStats, sp, mA, mB, nullptr, pair_grid(sp.n_items), st, nullptr, pdl && !timing));
    }

    sp.zero_n4 = 0;
    sp.idset = nullptr;
    // ---- u table, payload, (all-gather), weights, reductions, tau update ----
    mark(3, st);
    // table update + weights + local G_tau / loss terms + payload, one lane group per anchor
    a.n_blockpart = nblk;
    if (prof) a.dbg = dbg_buf + 2 * 2688 + 160 * 16;
    {
      cudaLaunchConfig_t cfg{};
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = (pdl && !timing) ? 1 : 0;
      cfg.gridDim = dim3(nblk, 1, 1);
      cfg.blockDim = dim3(kAnchorBlock, 1, 1);
      cfg.stream = st;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      FC_CUDA(cudaLaunchKernelEx(&cfg, fc::fc_anchor_kernel, a));
    }
    FC_CUDA(cudaGetLastError());
    if (K > 1) {
      // ONE all-gather carries u/tau/id, the v2 per-index tau gradients and the G_tau / loss
      // block partials of every rank (no scalar all-reduce, no second gather)
      if (use_peer && overlap2) {
        // payload + this rank's pass-2 parameters into every rank, on the gather stream beside
        // pass 2: pass 2 runs its own column tiles first (their parameters are this rank's, from
        // the per-anchor kernel) and waits for each rank's flag before that rank's columns
        fc::PeerGather g = pg_p[par];
        g.seq = seq;
        g.early_trigger = 0;
        g.wait_src = -1;
        FC_CUDA(cudaEventRecord(e_fork, st));
        FC_CUDA(cudaStreamWaitEvent(ws3, e_fork, 0));
        FC_CUDA(fc::launch_peer_gather(g, n_sm, kGatherThreads, ws3, false, true));
      } else if (use_peer) {
        // payload + this rank's pass-2 parameters into every rank (the u replica update of the
        // other ranks' ids follows on the side branch)
        fc::PeerGather g = pg_p[par];
        g.seq = seq;
        // pass 2 (programmatic launch) takes its SMs while the payload moves: its first tile's
        // operands and MMAs need only E; parameters are loaded after griddepcontrol.wait.
        // 128-thread blocks fit beside a pass-2 CTA's register file
        g.early_trigger = pdl && !timing ? 1 : 0;
        g.wait_src = -1;
        FC_CUDA(fc::launch_peer_gather(g, 128, 128, st));
      } else {
        FC_NCCL(ncclAllGather(send, recv, static_cast<size_t>(pstride), ncclFloat64, comm, st));
        a.weights_replica_only = 0;
        fc::fc_weights_kernel<<<(B + kWeightsBlock - 1) / kWeightsBlock, kWeightsBlock, 0, st>>>(a);
        FC_CUDA(cudaGetLastError());
      }
    }
    // the G_tau reduction, temperature step and IndividualTemp update only feed the next step
    // and the step scalars: they run on the side branch (after the payload gather)
    FC_CUDA(cudaEventRecord(side_fork, overlap2 ? ws3 : st));
    FC_CUDA(cudaStreamWaitEvent(ws2, side_fork, 0));
    fc::fc_reduce_kernel<<<1, 32, 0, ws2>>>(a);
    if (K > 1 && use_peer) {
      a.weights_replica_only = 1;
      fc::fc_weights_kernel<<<(B + kWeightsBlock - 1) / kWeightsBlock, kWeightsBlock, 0, ws2>>>(a);
    }
    if (indiv) fc::fc_indiv_update_kernel<<<(B + 255) / 256, 256, 0, ws2>>>(a);
    FC_CUDA(cudaGetLastError());
    FC_CUDA(cudaEventRecord(side_join, ws2));

    if (rs) {   // trainer.cpp:504-518: no weights for anchors of other ranks
      fc::fc_rs_mask_kernel<<<(B + 255) / 256, 256, 0, st>>>(a);
      FC_CUDA(cudaGetLastError());
    }
    if (test_delay_ns > 0) fc::fc_delay_kernel<<<1, 32, 0, st>>>(test_delay_ns);
    // ---- pass 2: Q' tiles (bf16) for both segments ----
    for (int s = 0; s < 2; ++s) {
      fc::SimSeg& g = sp.seg[s];
      g.row_stat = nullptr;
      g.partial = nullptr;
      const int off = rank * Bl;
      g.row_kappa = (s ? a.kap2 : a.kap1) + off;
      g.row_beta = (s ? a.bet2 : a.bet1) + off;
      g.row_coef = (s ? a.coef2 : a.coef1) + off;
      g.col_kappa = s ? a.kap1 : a.kap2;
      g.col_beta = s ? a.bet1 : a.bet2;
      g.col_coef = s ? a.coef1 : a.coef2;
      g.row_fac = (s ? a.fac2 : a.fac1) + off;
      g.col_fac = s ? a.fac1 : a.fac2;
      g.q = q + static_cast<size_t>(s) * Bl * ldq;
    }
    mark(4, st);
    if (shared_q) {   // K = 1: Q'_C = Q'_R^T -- one Q pass, the dE2 GEMM reads Q^T (MN-major A)
      sp.nseg = 1;
      sp.n_rb[1] = 0;
      sp.n_items = sp.n_rb[0] * n_jt;
    }
    if (prof) sp.dbg_out = dbg_buf + 2688;
    sp.q_factor = (!indiv && q_factor) ? 1 : 0;   // one shared temperature: single-exponential Q
    int p2_grid = pair_grid(sp.n_items);
    if (overlap2) {   // own column tiles first; a remote tile's parameters after its ranks' payload flags
      sp.local_first = 2;
      sp.col_lo = rank * Bl;
      sp.jt_lo = (rank * Bl + fc::kPairN - 1) / fc::kPairN;
      sp.n_loc = std::max(0, std::min((rank + 1) * Bl / fc::kPairN, n_jt) - sp.jt_lo);
      sp.rows_per_src = Bl;
      sp.src_flag = pg_p[par].my_flag;
      sp.abort_flag = pg_p[par].my_abort;
      sp.timeout_ns = pg_p[par].timeout_ns;
      sp.split_tail = 0;
      p2_grid = pair_grid(sp.n_items / 2);
      // the bounds: an own tile's columns are this rank's anchors (own slot final); the other
      // slots hold 0 or a peer's final values until its flag, so their max stays a valid bound
    }
    FC_CUDA(fc::launch_sim(fc::kSimQ, sp, mA, mB, mQo, p2_grid, st, nullptr, pdl && !timing));

    // ---- pass 2b: dE = c (Q' E - r o E_local) ----
    mark(5, st);
    fc::GemmParams gp{};
    gp.nseg = 2;
    gp.d = d;
    gp.n_nb = (d + fc::kGemmN - 1) / fc::kGemmN;
    gp.kb_total = ldq / fc::kBlockK;
    gp.scale = static_cast<float>(1.0 / (static_cast<double>(Bl) * static_cast<double>(B - 1)));
    gp.reset_at_exit = bnd;   // this parity's slots: the next writer is step t+2 (see e1g)
    gp.n_reset = K;
    if (prof) gp.dbg_out = dbg_buf + 2 * 2688;
    for (int s = 0; s < 2; ++s) {
      fc::GemmSeg& g = gp.seg[s];
      g.a_mn_major = (shared_q && s == 1) ? 1 : 0;
      g.rows = Bl;
      g.x_row0 = rank * Bl;
      g.r = rcoef;
      g.x = s ? E1 : E2;
      g.out = s ? out->de2 : out->de1;
      gp.n_mb[s] = (Bl + fc::kPairM - 1) / fc::kPairM;
    }
    gp.n_tiles = (gp.n_mb[0] + gp.n_mb[1]) * gp.n_nb;
    // every unit reduce-adds into dE (zeroed by pass 1 of this step): the GEMM's only
    // predecessor is pass 2, so its launch stays programmatic
    // persistent: exactly the clusters that co-reside (clusters of 4 pack into fewer than 148 SMs)
    const int gemm_ctas = (n_sm / 2) * 2;
    balance_units(gp, gemm_ctas / 2);
    CUtensorMap mX[2] = {mE2n, mE1n};
    CUtensorMap mQs[2] = {mQ[0], shared_q ? mQt : mQ[1]};
    if (out->de1 != map_o1 || out->de2 != map_o2) {
      const uint64_t rb = static_cast<uint64_t>(d) * 4;
      mO[0] = make_map(out->de1, d, Bl, rb, 32, 32, CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
      mO[1] = make_map(out->de2, d, Bl, rb, 32, 32, CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
      map_o1 = out->de1;
      map_o2 = out->de2;
    }
    FC_CUDA(fc::launch_gemm(pdl && !timing, gp, mQs, mX, mO, gemm_ctas, st));
    if (rs) enqueue_rs(out, E1, E2, st);
    mark(6, st);

    FC_CUDA(cudaStreamWaitEvent(st, side_join, 0));
    if (overlap) FC_CUDA(cudaStreamWaitEvent(st, e_join, 0));
  }

  // openclip_rs: this rank's anchors' contrast cotangents for every row of G (for_e1 = Q'_C^T E2[L],
  // for_e2 = Q'_R^T E1[L]: with the other anchors' weights zeroed, Q' column j of a non-local j holds
  // exactly engine.cpp:131-141's terms), minus its own rows (already in dE), reduce-scattered in
  // fp32 over NCCL, scaled by rs_shard_scale / K (engine.cpp:146-149 on the mean = sum / K).
  void enqueue_rs(fc_step_out* out, const __nv_bfloat16* E1, const __nv_bfloat16* E2, cudaStream_t st) {
    const size_t bd = static_cast<size_t>(B) * d, ld = static_cast<size_t>(Bl) * d;
    FC_CUDA(cudaMemsetAsync(rs_part, 0, 2 * bd * sizeof(float), st));
    fc::GemmParams gp{};
    gp.nseg = 2;
    gp.d = d;
    gp.n_nb = (d + fc::kGemmN - 1) / fc::kGemmN;
    gp.kb_total = Bl / fc::kBlockK;
    gp.scale = 1.0f;
    for (int s2 = 0; s2 < 2; ++s2) {
      fc::GemmSeg& g = gp.seg[s2];
      g.a_mn_major = 1;
      g.rows = B;
      g.x_row0 = 0;
      g.x_krow0 = rank * Bl;
      g.r = nullptr;
      g.x = s2 ? E1 : E2;
      g.out = rs_part + s2 * bd;
      gp.n_mb[s2] = (B + fc::kPairM - 1) / fc::kPairM;
    }
    gp.n_tiles = (gp.n_mb[0] + gp.n_mb[1]) * gp.n_nb;
    const int ctas = (n_sm / 2) * 2;
    balance_units(gp, ctas / 2);
    CUtensorMap mX[2] = {mE2n, mE1n};
    FC_CUDA(fc::launch_gemm(false, gp, mQtRS, mX, mPart, ctas, st));
    for (int s2 = 0; s2 < 2; ++s2)   // this rank's own rows: already in dE (local contrast terms)
      FC_CUDA(cudaMemsetAsync(rs_part + s2 * bd + static_cast<size_t>(rank) * ld, 0, ld * sizeof(float), st));
    FC_NCCL(ncclGroupStart());
    for (int s2 = 0; s2 < 2; ++s2)
      FC_NCCL(ncclReduceScatter(rs_part + s2 * bd, rs_shard + s2 * ld, ld, ncclFloat32, ncclSum, comm, st));
    FC_NCCL(ncclGroupEnd());
    const float c = static_cast<float>(1.0 / (static_cast<double>(Bl) * static_cast<double>(B - 1)));
    fc::fc_axpy2_kernel<<<std::min<long long>(4096, (ld + 255) / 256), 256, 0, st>>>(out->de1, out->de2, rs_shard,
                                                                                     rs_shard + ld, static_cast<long long>(ld), c);
    FC_CUDA(cudaGetLastError());
  }

  // The reference fabric's collectives of one step (trainer.cpp:422-425, 464, 479, 530-533, 572)
  // with its wire model (fabric.cpp:18-28), and this rank's actual peer bytes.
  void book_step() {
    if (K < 2) return;
    const unsigned long long k = static_cast<unsigned long long>(K), bl = static_cast<unsigned long long>(Bl);
    const unsigned long long ag = k * (k - 1), dd = static_cast<unsigned long long>(d);
    const bool mbcl = cfg.variant == FC_OPENCLIP_MBCL;
    const bool learn = cfg.variant == FC_FASTCLIP_V0 || cfg.variant == FC_FASTCLIP_V3 || mbcl;
    // E1 / E2 slices, bf16, to K - 1 peers
    book("feature-gather", 0, 2 * ag * bl * dd, 2 * (k - 1) * bl * dd * 2);
    if (!rs && !mbcl) book("u-gather", 0, ag * 2 * bl, (k - 1) * 2 * bl * 8);
    if (!rs && !mbcl && indiv) book("tau-gather", 0, ag * 2 * bl, (k - 1) * 2 * bl * 8);
    if (learn) book("tau-reduce", 1, 2 * (k - 1), use_peer ? (k - 1) * 3 * static_cast<unsigned long long>(nblk) * 8 : 8);
    if (rs) book("rs-grad", 2, 2 * ag * bl * dd, 2 * (k - 1) * bl * dd * 4);
    // what only the per-GPU replicas need: ids, the remaining payload columns, pass-2 parameters
    const unsigned long long payload = use_peer ? static_cast<unsigned long long>(pstride) * 8 + 8 * bl * 4 + 16
                                                : static_cast<unsigned long long>(pstride) * 8;
    unsigned long long used = 0;
    if (!rs && !mbcl) used += 2 * bl * 8 * (indiv ? 2 : 1);
    if (learn && use_peer) used += 3 * static_cast<unsigned long long>(nblk) * 8;
    book("replica-sync", 0, 0, (k - 1) * (payload > used ? payload - used : 0));
  }

  int kernels_per_step() const {
    int n = 1 /*prep*/ + 1 /*pass1*/ + 1 /*reduce*/ + (indiv ? 1 : 0) + 1 /*pass2*/ + 1 /*gemm*/;
    n += 1;   // fc_anchor_kernel
    if (K > 1) n += use_peer ? 3 /*two peer gathers + u replica*/ : 1 /*weights*/;
    if (rs) n += 3;   // weight mask, partial GEMM, axpy (+ NCCL's reduce-scatter kernel)
    return n;
  }

  void destroy() {
    // graphs first: NCCL keeps the communicator alive while a graph holds captured collectives
    cudaDeviceSynchronize();
    for (auto& g : graphs) {
      cudaGraphExecDestroy(g.exec);
      cudaGraphDestroy(g.graph);
    }
    graphs.clear();
    for (void* m : peer_maps) cudaIpcCloseMemHandle(m);
    peer_maps.clear();
    if (comm) {
      cudaDeviceSynchronize();
      ncclCommDestroy(comm);
    }
    for (void* p : {(void*)u1, (void*)u2, (void*)tau1, (void*)tau2, (void*)m1, (void*)v1, (void*)m2, (void*)v2,
                    (void*)s1, (void*)s2, (void*)tau_state, (void*)e1g, (void*)e2g, (void*)diag, (void*)rowstat,
                    (void*)partial, (void*)col_partial, (void*)clamps, (void*)bounds, (void*)f64, (void*)red, (void*)par, (void*)rcoef,
                    (void*)q, (void*)err, (void*)pflags, (void*)ptickets, (void*)idset,
                    (void*)step_tag, (void*)rs_part, (void*)rs_shard})
      if (p) cudaFree(p);
    if (recv && recv != send) cudaFree(recv);
    if (send) cudaFree(send);
    if (result_h) cudaFreeHost(result_h);
    if (scal) cudaFree(scal);
    if (ws) cudaStreamDestroy(ws);
    if (ws2) cudaStreamDestroy(ws2);
    if (ws3) cudaStreamDestroy(ws3);
    if (e_fork) cudaEventDestroy(e_fork);
    if (e_join) cudaEventDestroy(e_join);
    cudaEventDestroy(side_fork);
    cudaEventDestroy(side_join);
    cudaEventDestroy(done);
    cudaEventDestroy(fork);
    for (auto& e : ev) cudaEventDestroy(e);
    ev.clear();
  }
};

template <class Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return FC_OK;
  } catch (const FcError& e) {
    g_last_error = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return FC_ERR_CUDA;
  }
}

// ---- the reference's binary formats (state.cpp:11-33, :73-95, :133-162; checkpoint.cpp:9-114) ----
// Vectors are int64 length + doubles; ScalarAdam is {double m, double v, long long step}; FCK1 is the
// field sequence of write_checkpoint. Tables are staged through host memory.
struct BinOut {
  std::ofstream os;
  explicit BinOut(const char* path) : os(path, std::ios::binary | std::ios::trunc) {
    if (!os) throw FcError{FC_ERR_IO, std::string("cannot open '") + path + "' for writing"};
  }
  void raw(const void* p, size_t n) { os.write(static_cast<const char*>(p), static_cast<std::streamsize>(n)); }
  template <class T> void pod(const T& v) { raw(&v, sizeof(T)); }
  void vec(const double* p, int64_t n) {
    pod(n);
    raw(p, sizeof(double) * static_cast<size_t>(n));
  }
  void check() {
    if (!os) throw FcError{FC_ERR_IO, "write failed"};
  }
};
struct BinIn {
  std::ifstream is;
  explicit BinIn(const char* path) : is(path, std::ios::binary) {
    if (!is) throw FcError{FC_ERR_IO, std::string("cannot open '") + path + "'"};
  }
  void raw(void* p, size_t n) {
    is.read(static_cast<char*>(p), static_cast<std::streamsize>(n));
    if (!is) throw FcError{FC_ERR_IO, "truncated stream"};
  }
  template <class T> T pod() {
    T v;
    raw(&v, sizeof(T));
    return v;
  }
  std::vector<double> vec() {
    const int64_t n = pod<int64_t>();
    if (n < 0) throw FcError{FC_ERR_IO, "negative vector length"};
    std::vector<double> v(static_cast<size_t>(n));
    raw(v.data(), sizeof(double) * v.size());
    return v;
  }
};

// UTable::write (state.cpp:73-76) + IndividualTemp::write (state.cpp:133-144) of a context.
void write_tables(LossStep* s, BinOut& o) {
  FC_CUDA(cudaDeviceSynchronize());
  const size_t n = static_cast<size_t>(s->cfg.n_train);
  std::vector<double> h(n);
  for (double* t : {s->u1, s->u2}) {
    FC_CUDA(cudaMemcpy(h.data(), t, n * 8, cudaMemcpyDeviceToHost));
    o.vec(h.data(), static_cast<int64_t>(n));
  }
}
void write_individual(LossStep* s, BinOut& o) {
  const size_t n = static_cast<size_t>(s->cfg.n_train);
  std::vector<double> h(n);
  for (double* t : {s->tau1, s->tau2}) {
    FC_CUDA(cudaMemcpy(h.data(), t, n * 8, cudaMemcpyDeviceToHost));
    o.vec(h.data(), static_cast<int64_t>(n));
  }
  o.pod(s->cfg.tau0);
  std::vector<double> m(n), v(n);
  std::vector<long long> st(n);
  std::vector<uint8_t> aos(n * 24);   // ScalarAdam records, AoS (state.cpp:137-143)
  for (int t = 0; t < 2; ++t) {
    FC_CUDA(cudaMemcpy(m.data(), t ? s->m2 : s->m1, n * 8, cudaMemcpyDeviceToHost));
    FC_CUDA(cudaMemcpy(v.data(), t ? s->v2 : s->v1, n * 8, cudaMemcpyDeviceToHost));
    FC_CUDA(cudaMemcpy(st.data(), t ? s->s2 : s->s1, n * 8, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < n; ++i) {
      std::memcpy(&aos[24 * i], &m[i], 8);
      std::memcpy(&aos[24 * i + 8], &v[i], 8);
      std::memcpy(&aos[24 * i + 16], &st[i], 8);
    }
    o.raw(aos.data(), aos.size());
  }
}
// UTable::read (state.cpp:87-95) + IndividualTemp::read (state.cpp:146-162) into a context.
void read_tables(LossStep* s, BinIn& in) {
  const size_t n = static_cast<size_t>(s->cfg.n_train);
  const std::vector<double> a = in.vec(), b = in.vec();
  if (a.size() != b.size()) throw FcError{FC_ERR_IO, "UTable: track lengths differ"};
  if (a.size() != n) throw FcError{FC_ERR_SHAPE, "UTable::load: size mismatch with n_train"};
  FC_CUDA(cudaDeviceSynchronize());
  FC_CUDA(cudaMemcpy(s->u1, a.data(), n * 8, cudaMemcpyHostToDevice));
  FC_CUDA(cudaMemcpy(s->u2, b.data(), n * 8, cudaMemcpyHostToDevice));
}
void read_individual(LossStep* s, BinIn& in) {
  const size_t n = static_cast<size_t>(s->cfg.n_train);
  const std::vector<double> t1 = in.vec(), t2 = in.vec();
  if (t1.size() != t2.size()) throw FcError{FC_ERR_IO, "IndividualTemp: track lengths differ"};
  if (t1.size() != n) throw FcError{FC_ERR_SHAPE, "IndividualTemp: size mismatch with n_train"};
  const double tau0 = in.pod<double>();
  if (tau0 != s->cfg.tau0) throw FcError{FC_ERR_CONFIG, "IndividualTemp: tau0 differs from temperature.tau0"};
  std::vector<uint8_t> aos(n * 24);
  std::vector<double> m(n), v(n);
  std::vector<long long> st(n);
  FC_CUDA(cudaDeviceSynchronize());
  FC_CUDA(cudaMemcpy(s->tau1, t1.data(), n * 8, cudaMemcpyHostToDevice));
  FC_CUDA(cudaMemcpy(s->tau2, t2.data(), n * 8, cudaMemcpyHostToDevice));
  for (int t = 0; t < 2; ++t) {
    in.raw(aos.data(), aos.size());
    for (size_t i = 0; i < n; ++i) {
      std::memcpy(&m[i], &aos[24 * i], 8);
      std::memcpy(&v[i], &aos[24 * i + 8], 8);
      std::memcpy(&st[i], &aos[24 * i + 16], 8);
    }
    FC_CUDA(cudaMemcpy(t ? s->m2 : s->m1, m.data(), n * 8, cudaMemcpyHostToDevice));
    FC_CUDA(cudaMemcpy(t ? s->v2 : s->v1, v.data(), n * 8, cudaMemcpyHostToDevice));
    FC_CUDA(cudaMemcpy(t ? s->s2 : s->s1, st.data(), n * 8, cudaMemcpyHostToDevice));
  }
}

constexpr uint32_t kFck1Magic = 0x46434b31;   // "FCK1" (checkpoint.cpp:9)

}  // namespace

extern "C" {

const char* fc_last_error(void) { return g_last_error.c_str(); }

int fc_config_defaults(int32_t variant, int64_t n_train, fc_config* out) {
  if (!out) return FC_ERR_SHAPE;
  if (variant < 0 || variant > 6) {
    g_last_error = "unknown variant";
    return FC_ERR_CONFIG;
  }
  std::memset(out, 0, sizeof(*out));
  out->variant = variant;
  out->n_train = n_train;
  // trainer.cpp:139-194 with the registry defaults of config.cpp:36-60
  out->tau_init = variant == FC_FASTCLIP_V3 ? 0.07 : 0.03;
  out->tau0 = 0.005;
  if (variant == FC_SOGCLR || variant == FC_FASTCLIP_V1) out->tau_lr = 0.0;
  else if (is_individual(variant)) out->tau_lr = 1e-2;
  else out->tau_lr = 2e-4;
  out->rho = is_individual(variant) ? 9.0 : (variant == FC_FASTCLIP_V3 ? 6.5 : 0.0);
  out->beta1 = 0.9;
  out->beta2 = 0.999;
  out->adam_eps = 1e-8;
  out->lr_decay_enabled = variant == FC_FASTCLIP_V3 ? 1 : 0;
  out->lr_decay_threshold = 0.03;
  out->lr_decay_factor = 1.0 / 3.0;
  out->scale_by_tau = (variant == FC_FASTCLIP_V0 || variant == FC_OPENCLIP_MBCL) ? 0 : 1;
  out->world = 1;
  out->reduction = variant == FC_OPENCLIP_MBCL ? 1 : 0;   // fabric.reduction = auto (trainer.cpp:86-88)
  return FC_OK;
}

double fc_gamma_at(int32_t cosine, double constant, double gamma_min, int64_t decay_epochs, int64_t iters_per_epoch,
                   int64_t t) {
  // schedules.cpp:25-31
  if (!cosine) return constant;
  const int64_t epoch = t / iters_per_epoch;
  if (epoch >= decay_epochs) return gamma_min;
  const double frac = static_cast<double>(epoch) / static_cast<double>(decay_epochs);
  return 0.5 * (1.0 + std::cos(3.141592653589793238462643383279502884 * frac)) * (1.0 - gamma_min) + gamma_min;
}

double fc_epsilon_at(double initial, double late, int64_t switch_epoch, int64_t epoch) {
  if (switch_epoch < 0) return initial;  // schedules.cpp:62-65
  return epoch < switch_epoch ? initial : late;
}

// opt::temperature_step (optimizers.cpp:77-83): scalar_adamw_step with weight decay 0
// (optimizers.cpp:65-75: bias correction with step + 1, then ++step) and the projection
// max(tau, tau0). Host scalar, the same arithmetic as the device finalize_step.
int fc_temperature_step(double* m, double* v, int64_t* step, double tau, double grad, double lr, double beta1,
                        double beta2, double eps, double tau0, double* tau_out) {
  if (!m || !v || !step || !tau_out) return FC_ERR_SHAPE;
  if (!std::isfinite(grad)) {
    g_last_error = "temperature_step: non-finite gradient (NumericError, optimizers.cpp:67)";
    return FC_ERR_NUMERIC;
  }
  *m = beta1 * *m + (1.0 - beta1) * grad;
  *v = beta2 * *v + (1.0 - beta2) * grad * grad;
  const double c1 = 1.0 - std::pow(beta1, static_cast<double>(*step + 1));
  const double c2 = 1.0 - std::pow(beta2, static_cast<double>(*step + 1));
  *step += 1;
  const double r = (*m / c1) / (std::sqrt(*v / c2) + eps);
  const double next = tau - lr * (r + 0.0 * tau);
  *tau_out = next < tau0 ? tau0 : next;
  return FC_OK;
}

// UTable::update + snapshot (state.cpp:45-71) on device tables: u <- (1 - gamma) u + gamma g at
// ids[0..count), then the post-update values in batch order.
__global__ void fc_table_update_kernel(double* u1, double* u2, int64_t n, const int32_t* ids, const double* g1,
                                       const double* g2, int count, double gamma, double* o1, double* o2,
                                       int32_t* status) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= count) return;
  const int id = ids[r];
  if (id < 0 || id >= n) {   // ShapeError (state.cpp:46)
    if (status) atomicExch(status, FC_ERR_SHAPE);
    return;
  }
  const double a = g1[r], b = g2[r];
  if (a < 0.0 || b < 0.0) {   // domain_error (state.cpp:51)
    if (status) atomicExch(status, FC_ERR_DOMAIN);
    return;
  }
  const double x1 = (1.0 - gamma) * u1[id] + gamma * a;
  const double x2 = (1.0 - gamma) * u2[id] + gamma * b;
  u1[id] = x1;
  u2[id] = x2;
  if (o1) o1[r] = x1;
  if (o2) o2[r] = x2;
}

int fc_table_update(double* u1, double* u2, int64_t n_train, const int32_t* ids, const double* g1, const double* g2,
                    int32_t count, double gamma, double* u1_out, double* u2_out, int32_t* status, void* stream) {
  return guarded([&] {
    if (!(gamma > 0.0) || gamma > 1.0) throw FcError{FC_ERR_DOMAIN, "gamma must be in (0,1] (state.cpp:50)"};
    if (!u1 || !u2 || !ids || !g1 || !g2 || count < 0) throw FcError{FC_ERR_SHAPE, "table_update: bad arguments"};
    if (count == 0) return;
    fc_table_update_kernel<<<(count + 255) / 256, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        u1, u2, n_train, ids, g1, g2, count, gamma, u1_out, u2_out, status);
    FC_CUDA(cudaGetLastError());
  });
}

// engine::grad_tau_unscaled (v0, engine.cpp:208-224), grad_tau_margin (v3, :226-238),
// grad_tau_mbcl (:261-266) -> gtau[0] (this worker's G_tau,k, before the mean all-reduce), and
// grad_tau_individual (v2 / iSogCLR, :240-259) -> gt1/gt2 per local anchor. One block,
// fixed-order fp64 reduction (deterministic).
__global__ void fc_grad_tau_kernel(int variant, int count, long long batch, const double* u1, const double* u2,
                                   const double* ds1, const double* ds2, const double* t1, const double* t2, double eps,
                                   double rho, double tau, long long n_train, double* gtau, double* gt1, double* gt2) {
  __shared__ double sh[2][32];
  const bool indiv = variant == FC_ISOGCLR || variant == FC_FASTCLIP_V2;
  const double e = variant == FC_OPENCLIP_MBCL ? 1.0 / static_cast<double>(batch - 1) : eps;
  double a = 0.0, b = 0.0;
  for (int r = threadIdx.x; r < count; r += blockDim.x) {
    if (indiv) {
      const double inv_n = 1.0 / static_cast<double>(n_train);
      gt1[r] = inv_n * (log(eps + u1[r]) + rho + t1[r] * ds1[r] / (eps + u1[r]));
      gt2[r] = inv_n * (log(eps + u2[r]) + rho + t2[r] * ds2[r] / (eps + u2[r]));
    } else {
      a += ds1[r] / (e + u1[r]) + ds2[r] / (e + u2[r]);
      b += log(eps + u1[r]) + log(eps + u2[r]);
    }
  }
  if (indiv) return;
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  if ((threadIdx.x & 31) == 0) { sh[0][threadIdx.x >> 5] = a; sh[1][threadIdx.x >> 5] = b; }
  __syncthreads();
  if (threadIdx.x != 0) return;
  a = 0.0; b = 0.0;
  for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) { a += sh[0][w]; b += sh[1][w]; }
  const double unscaled = a / static_cast<double>(count);
  *gtau = variant == FC_FASTCLIP_V3 ? b / static_cast<double>(count) + 2.0 * rho + tau * unscaled : unscaled;
}

int fc_grad_tau(int32_t variant, int32_t count, int64_t batch, const double* u1, const double* u2, const double* dsum1,
                const double* dsum2, const double* t1, const double* t2, double eps, double rho, double tau,
                int64_t n_train, double* gtau, double* gt1, double* gt2, void* stream) {
  return guarded([&] {
    if (variant < 0 || variant > 6) throw FcError{FC_ERR_CONFIG, "unknown variant"};
    if (variant == FC_SOGCLR || variant == FC_FASTCLIP_V1) throw FcError{FC_ERR_CONFIG, "constant-tau variant has no tau gradient"};
    if (count < 1 || batch < 2) throw FcError{FC_ERR_DEGENERATE_BATCH, "grad_tau: empty slice or batch < 2"};
    const bool indiv = variant == FC_ISOGCLR || variant == FC_FASTCLIP_V2;
    if (!u1 || !u2 || !dsum1 || !dsum2 || (indiv && (!t1 || !t2 || !gt1 || !gt2 || n_train < 2)) || (!indiv && !gtau))
      throw FcError{FC_ERR_SHAPE, "grad_tau: null pointer / n_train"};
    if (eps < 0.0) throw FcError{FC_ERR_DOMAIN, "epsilon must be non-negative"};
    fc_grad_tau_kernel<<<1, 1024, 0, static_cast<cudaStream_t>(stream)>>>(variant, count, batch, u1, u2, dsum1, dsum2, t1, t2,
                                                                          eps, rho, tau, n_train, gtau, gt1, gt2);
    FC_CUDA(cudaGetLastError());
  });
}

int fc_nccl_unique_id(uint8_t out[128]) {
  return guarded([&] {
    ncclUniqueId id;
    FC_NCCL(ncclGetUniqueId(&id));
    std::memcpy(out, &id, sizeof(id));
  });
}

int fc_create(const fc_config* cfg, void** ctx) {
  if (!cfg || !ctx) return FC_ERR_SHAPE;
  auto* s = new LossStep;
  const int rc = guarded([&] { s->init(cfg); });
  if (rc != FC_OK) {
    s->destroy();
    delete s;
    *ctx = nullptr;
    return rc;
  }
  *ctx = s;
  return FC_OK;
}

int fc_destroy(void* ctx) {
  if (!ctx) return FC_OK;
  auto* s = static_cast<LossStep*>(ctx);
  s->destroy();
  delete s;
  return FC_OK;
}

int fc_loss_step(void* ctx, const fc_step_in* in, fc_step_out* out, void* stream) {
  if (!ctx) return FC_ERR_SHAPE;
  return guarded([&] { static_cast<LossStep*>(ctx)->step(in, out, static_cast<cudaStream_t>(stream)); });
}

int fc_step_scalars_get(void* ctx, fc_step_scalars* out) {
  if (!ctx || !out) return FC_ERR_SHAPE;
  auto* s = static_cast<LossStep*>(ctx);
  int rc = guarded([&] { FC_CUDA(cudaEventSynchronize(s->done)); });
  if (rc != FC_OK) return rc;
  out->loss = s->result_h->loss;
  out->gtau = s->result_h->gtau;
  out->tau = s->result_h->tau;
  out->exp_clamps = s->result_h->clamps;
  out->latched = s->result_h->latched;
  if (const int e = s->result_h->err) {   // device-detected failures of the step (sticky)
    g_last_error = e == FC_ERR_SHAPE ? "ids: dataset index out of range [0, n_train) (UTable::update, state.cpp:46)"
                 : e == FC_ERR_NUMERIC ? "non-finite temperature gradient (optimizers.cpp:67)"
                 : e == FC_ERR_OWNERSHIP ? "ids: a dataset index appears twice in this rank's batch; no u/tau entry "
                                           "of the step was written (OwnershipViolation, state.cpp:47-49)"
                 : e == FC_ERR_COLLECTIVE_ABORTED ? "peer gather aborted: a rank stopped stepping or timed out "
                                                    "(CollectiveAborted, fabric.cpp:228-235)"
                 : "device-side step failure";
    return e;
  }
  return FC_OK;
}

int fc_local_views(void* ctx, double* g1, double* g2, double* u1, double* u2, double* t1, double* t2) {
  if (!ctx) return FC_ERR_SHAPE;
  auto* s = static_cast<LossStep*>(ctx);
  return guarded([&] {
    FC_CUDA(cudaEventSynchronize(s->done));
    const size_t n = static_cast<size_t>(s->Bl) * 8;
    double* host[6] = {g1, g2, u1, u2, t1, t2};
    const double* dev[6] = {s->args.g1, s->args.g2, s->args.u1, s->args.u2, s->args.t_loc1, s->args.t_loc2};
    for (int i = 0; i < 6; ++i)
      if (host[i]) FC_CUDA(cudaMemcpy(host[i], dev[i], n, cudaMemcpyDeviceToHost));
  });
}

int fc_table_download(void* ctx, double* u1, double* u2, double* tau1, double* tau2, double* m1, double* v1,
                      int64_t* s1, double* m2, double* v2, int64_t* s2) {
  if (!ctx) return FC_ERR_SHAPE;
  auto* s = static_cast<LossStep*>(ctx);
  return guarded([&] {
    FC_CUDA(cudaDeviceSynchronize());
    const size_t n = static_cast<size_t>(s->cfg.n_train) * 8;
    if (u1) FC_CUDA(cudaMemcpy(u1, s->u1, n, cudaMemcpyDeviceToHost));
    if (u2) FC_CUDA(cudaMemcpy(u2, s->u2, n, cudaMemcpyDeviceToHost));
    if (s->indiv) {
      void* host[8] = {tau1, tau2, m1, v1, s1, m2, v2, s2};
      const void* dev[8] = {s->tau1, s->tau2, s->m1, s->v1, s->s1, s->m2, s->v2, s->s2};
      for (int i = 0; i < 8; ++i)
        if (host[i]) FC_CUDA(cudaMemcpy(host[i], dev[i], n, cudaMemcpyDeviceToHost));
    }
  });
}

int fc_table_upload(void* ctx, const double* u1, const double* u2, const double* tau1, const double* tau2,
                    const double* m1, const double* v1, const int64_t* s1, const double* m2, const double* v2,
                    const int64_t* s2) {
  if (!ctx) return FC_ERR_SHAPE;
  auto* s = static_cast<LossStep*>(ctx);
  return guarded([&] {
    FC_CUDA(cudaDeviceSynchronize());
    const size_t n = static_cast<size_t>(s->cfg.n_train) * 8;
    if (u1) FC_CUDA(cudaMemcpy(s->u1, u1, n, cudaMemcpyHostToDevice));
    if (u2) FC_CUDA(cudaMemcpy(s->u2, u2, n, cudaMemcpyHostToDevice));
    if (s->indiv) {
      const void* host[8] = {tau1, tau2, m1, v1, s1, m2, v2, s2};
      void* dev[8] = {s->tau1, s->tau2, s->m1, s->v1, s->s1, s->m2, s->v2, s->s2};
      for (int i = 0; i < 8; ++i)
        if (host[i]) FC_CUDA(cudaMemcpy(dev[i], host[i], n, cudaMemcpyHostToDevice));
    }
  });
}

int fc_tau_state_get(void* ctx, double* tau, double* m, double* v, int64_t* step, int32_t* latched) {
  if (!ctx) return FC_ERR_SHAPE;
  auto* s = static_cast<LossStep*>(ctx);
  return guarded([&] {
    fc::TauState ts;
    FC_CUDA(cudaDeviceSynchronize());
    FC_CUDA(cudaMemcpy(&ts, s->tau_state, sizeof(ts), cudaMemcpyDeviceToHost));
    if (tau) *tau = ts.tau;
    if (m) *m = ts.m;
    if (v) *v = ts.v;
    if (step) *step = ts.step;
    if (latched) *latched = ts.latched;
  });
}

int fc_tau_state_set(void* ctx, double tau, double m, double v, int64_t step, int32_t latched) {
  if (!ctx) return FC_ERR_SHAPE;
  auto* s = static_cast<LossStep*>(ctx);
  return guarded([&] {
    fc::TauState ts{tau, m, v, static_cast<long long>(step), latched, 0};
    FC_CUDA(cudaDeviceSynchronize());
    FC_CUDA(cudaMemcpy(s->tau_state, &ts, sizeof(ts), cudaMemcpyHostToDevice));
  });
}

int fc_set_phase_timing(void* ctx, int32_t slots) {
  if (!ctx) return FC_ERR_SHAPE;
  auto* s = static_cast<LossStep*>(ctx);
  return guarded([&] {
    FC_CUDA(cudaDeviceSynchronize());
    for (auto& e : s->ev) cudaEventDestroy(e);
    s->ev.clear();
    s->ev_slots = slots > 0 ? slots : 0;
    s->ev.resize(static_cast<size_t>(s->ev_slots) * (LossStep::kPhases + 1));
    for (auto& e : s->ev) FC_CUDA(cudaEventCreate(&e));
    s->ev_cur = 0;
    s->ev_last = 0;
    s->timing = s->ev_slots > 0;
  });
}

int fc_phase_times(void* ctx, int32_t slot, float* ms, int32_t n) {
  if (!ctx || !ms) return FC_ERR_SHAPE;
  auto* s = static_cast<LossStep*>(ctx);
  return guarded([&] {
    if (s->ev_slots == 0) throw FcError{FC_ERR_CONFIG, "phase timing not enabled"};
    const int k = slot < 0 ? s->ev_last : slot % s->ev_slots;
    cudaEvent_t* e = s->ev.data() + static_cast<size_t>(k) * (LossStep::kPhases + 1);
    FC_CUDA(cudaEventSynchronize(e[LossStep::kPhases]));
    for (int i = 0; i < n && i < LossStep::kPhases; ++i) FC_CUDA(cudaEventElapsedTime(&ms[i], e[i], e[i + 1]));
  });
}

int fc_debug_reset(void* ctx) {   // debug timeline: prep first-entry (min) / last-exit (max) slots
  if (!ctx) return FC_ERR_SHAPE;
  auto* s = static_cast<LossStep*>(ctx);
  return guarded([&] {
    FC_CUDA(cudaDeviceSynchronize());
    if (s->dbg_buf) {
      long long* slot = s->dbg_buf + 2 * 2688 + 160 * 16 + 8 * 640;
      FC_CUDA(cudaMemset(slot, 0xff, 8));
      FC_CUDA(cudaMemset(slot + 1, 0, 8));
    }
  });
}

int fc_debug_counters(void* ctx, long long* out /* host [2*128*8] */) {
  if (!ctx) return FC_ERR_SHAPE;
  auto* s = static_cast<LossStep*>(ctx);
  return guarded([&] {
    FC_CUDA(cudaDeviceSynchronize());
    if (s->dbg_buf) FC_CUDA(cudaMemcpy(out, s->dbg_buf, (2 * 2688 + 160 * 16 + 8192) * 8, cudaMemcpyDeviceToHost));
  });
}

int fc_kernels_per_step(void* ctx) { return ctx ? static_cast<LossStep*>(ctx)->kernels_per_step() : 0; }

int fc_debug_similarity(const void* a, const void* b, int32_t rows, int32_t cols, int32_t dim, float* out,
                        void* stream) {
  return guarded([&] {
    if (dim % 8 != 0) throw FcError{FC_ERR_UNSUPPORTED, "dim % 8"};
    const uint64_t rb = static_cast<uint64_t>(dim) * 2;
    CUtensorMap ma = make_map(a, dim, rows, rb, 64, 128);
    CUtensorMap mb = make_map(b, dim, cols, rb, 64, 128);
    fc::SimParams sp{};
    sp.nseg = 1;
    sp.d = dim;
    sp.n_jt = (cols + fc::kPairN - 1) / fc::kPairN;
    sp.n_rb[0] = (rows + fc::kPairM - 1) / fc::kPairM;
    sp.n_rb[1] = 0;
    sp.seg[0].rows = rows;
    sp.seg[0].a_row0 = 0;
    sp.seg[0].cols = cols;
    sp.n_items = sp.n_rb[0] * sp.n_jt;
    static float* dbg_bounds = nullptr;
    if (!dbg_bounds) {
      dbg_bounds = dalloc<float>(4);
      const float big[4] = {1e30f, 1e30f, 1e30f, 0.f};
      FC_CUDA(cudaMemcpy(dbg_bounds, big, sizeof(big), cudaMemcpyHostToDevice));
    }
    sp.bounds = dbg_bounds;
    sp.n_bounds = 1;
    int dev = 0;
    cudaGetDevice(&dev);
    FC_CUDA(fc::sim_set_smem());
    const int pairs = std::min(sm_count(dev) / 2, sp.n_items);
    FC_CUDA(fc::launch_sim(fc::kSimRaw, sp, &ma, &mb, nullptr, std::max(1, pairs) * 2, static_cast<cudaStream_t>(stream), out));
  });
}

// engine::g_values (engine.cpp:151-176) and engine::dtau_sums (engine.cpp:182-204) for the
// local slice [local_begin, local_begin + local_count) of a global batch, on the step's pass-1
// kernel (segments R = S[L,G] and C = S^T[L,G], safe_exp in the log2 domain). Stateless:
// workspaces come from the stream-ordered allocator and are released on the same stream.
int fc_g_values(const void* e1g, const void* e2g, int32_t batch, int32_t dim, const double* t1_local,
                const double* t2_local, int32_t local_begin, int32_t local_count, double* g1, double* g2,
                double* dsum1, double* dsum2, uint64_t* clamps, void* stream) {
  return guarded([&] {
    if (batch < 2) throw FcError{FC_ERR_DEGENERATE_BATCH, "g_values: global batch must have >= 2 pairs"};
    if (local_begin < 0 || local_count <= 0 || local_begin + local_count > batch)
      throw FcError{FC_ERR_SHAPE, "g_values: local slice outside the global batch"};
    if (dim < 8 || dim % 8 != 0) throw FcError{FC_ERR_UNSUPPORTED, "dim must be a positive multiple of 8"};
    if (!e1g || !e2g || !t1_local || !t2_local || !g1 || !g2 || (!dsum1) != (!dsum2))
      throw FcError{FC_ERR_SHAPE, "g_values: null pointer"};
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int B = batch, d = dim, lo = local_begin, cnt = local_count;
    const int n_jt = (B + fc::kPairN - 1) / fc::kPairN;
    const int nparts = n_jt * 4;
    const size_t part_bytes = static_cast<size_t>(cnt) * nparts * sizeof(float2);
    uint8_t* ws = nullptr;
    const size_t ws_bytes = 2 * part_bytes + 2 * cnt * sizeof(float2) + 64;
    FC_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ws), ws_bytes, st));
    float2* pR = reinterpret_cast<float2*>(ws);
    float2* pC = reinterpret_cast<float2*>(ws + part_bytes);
    float2* rsR = reinterpret_cast<float2*>(ws + 2 * part_bytes);
    float2* rsC = rsR + cnt;
    float* bnd = reinterpret_cast<float*>(rsC + cnt);
    unsigned long long* ncl = reinterpret_cast<unsigned long long*>(bnd + 4);
    FC_CUDA(cudaMemsetAsync(bnd, 0, 4 * sizeof(float) + sizeof(unsigned long long), st));
    fc::fc_rows_kernel<<<(B * 32 + 127) / 128, 128, 0, st>>>(static_cast<const __nv_bfloat16*>(e1g),
                                                            static_cast<const __nv_bfloat16*>(e2g), B, d, lo, cnt,
                                                            t1_local, t2_local, rsR, rsC, bnd, nullptr);
    FC_CUDA(cudaGetLastError());
    const uint64_t rb = static_cast<uint64_t>(d) * 2;
    CUtensorMap m1 = make_map(e1g, d, B, rb, 64, 128), m2 = make_map(e2g, d, B, rb, 64, 128);
    fc::SimParams sp{};
    sp.nseg = 2;
    sp.d = d;
    sp.n_jt = n_jt;
    for (int s = 0; s < 2; ++s) {
      fc::SimSeg& g = sp.seg[s];
      g.rows = cnt;
      g.a_row0 = lo;
      g.cols = B;
      g.row_stat = s ? rsC : rsR;
      g.partial = s ? pC : pR;
      sp.n_rb[s] = (cnt + fc::kPairM - 1) / fc::kPairM;
    }
    sp.n_items = (sp.n_rb[0] + sp.n_rb[1]) * n_jt;
    sp.clamps = ncl;
    sp.bounds = bnd;
    sp.n_bounds = 1;
    int dev = 0;
    FC_CUDA(cudaGetDevice(&dev));
    FC_CUDA(fc::sim_set_smem());   // per-device function attribute: set on the current device every call
    CUtensorMap mA[2] = {m1, m2}, mB[2] = {m2, m1};
    const int pairs = std::max(1, std::min(sm_count(dev) / 2, sp.n_items));
    FC_CUDA(fc::launch_sim(fc::kSimStats, sp, mA, mB, nullptr, pairs * 2, st, nullptr));
    fc::fc_gsum_kernel<<<(cnt + 127) / 128, 128, 0, st>>>(pR, pC, nparts, cnt, B, rsR, rsC, t1_local, t2_local, g1, g2,
                                                         dsum1, dsum2);
    FC_CUDA(cudaGetLastError());
    if (clamps) FC_CUDA(cudaMemcpyAsync(clamps, ncl, sizeof(uint64_t), cudaMemcpyDeviceToDevice, st));
    FC_CUDA(cudaFreeAsync(ws, st));
  });
}

// engine::embedding_cotangents (engine.cpp:77-121) for the local slice [local_begin,
// local_begin + local_count) of a global batch with the caller's PairWeights (w, t over G):
// pass 1 (row sums for r_i), the pass-2 Q' tiles of both segments (two-exponential path, t per
// anchor) and the weighted-gradient GEMM -- the step's kernels on caller-provided operands.
// Stateless: workspaces come from the stream-ordered allocator.
int fc_embedding_cotangents(const void* e1g, const void* e2g, int32_t batch, int32_t dim, const double* w1,
                            const double* w2, const double* t1, const double* t2, int32_t local_begin,
                            int32_t local_count, float* de1, float* de2, void* stream) {
  return guarded([&] {
    if (batch < 2) throw FcError{FC_ERR_DEGENERATE_BATCH, "embedding_cotangents: global batch must have >= 2 pairs"};
    if (local_begin < 0 || local_count <= 0 || local_begin + local_count > batch)
      throw FcError{FC_ERR_SHAPE, "embedding_cotangents: local slice outside the global batch"};
    if (dim < 8 || dim % 8 != 0) throw FcError{FC_ERR_UNSUPPORTED, "dim must be a positive multiple of 8"};
    if (!e1g || !e2g || !w1 || !w2 || !t1 || !t2 || !de1 || !de2)
      throw FcError{FC_ERR_SHAPE, "embedding_cotangents: null pointer"};
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int B = batch, d = dim, lo = local_begin, cnt = local_count;
    const int n_jt = (B + fc::kPairN - 1) / fc::kPairN, nparts = n_jt * 4;
    const int ldq = (B + 63) / 64 * 64;
    const size_t np = static_cast<size_t>(n_jt) * fc::kPairN;
    // workspace: partials, row stats, diag, 8 parameter arrays, r, bounds + clamps, Q'
    const size_t part_b = static_cast<size_t>(cnt) * nparts * sizeof(float2);
    const size_t q_b = 2 * static_cast<size_t>(cnt) * ldq * 2;
    const size_t off_rs = 2 * part_b, off_diag = off_rs + 2 * cnt * sizeof(float2);
    const size_t off_par = (off_diag + B * sizeof(float) + 255) / 256 * 256;
    const size_t off_r = off_par + 8 * np * sizeof(float);
    const size_t off_b = (off_r + cnt * sizeof(float) + 255) / 256 * 256;
    const size_t off_q = off_b + 256;
    uint8_t* ws = nullptr;
    FC_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&ws), off_q + q_b, st));
    float2* pR = reinterpret_cast<float2*>(ws);
    float2* pC = reinterpret_cast<float2*>(ws + part_b);
    float2* rsR = reinterpret_cast<float2*>(ws + off_rs);
    float2* rsC = rsR + cnt;
    float* diag = reinterpret_cast<float*>(ws + off_diag);
    float* par = reinterpret_cast<float*>(ws + off_par);
    float* rco = reinterpret_cast<float*>(ws + off_r);
    float* bnd = reinterpret_cast<float*>(ws + off_b);
    unsigned long long* ncl = reinterpret_cast<unsigned long long*>(bnd + 4);
    __nv_bfloat16* q = reinterpret_cast<__nv_bfloat16*>(ws + off_q);
    FC_CUDA(cudaMemsetAsync(par, 0, 8 * np * sizeof(float), st));   // zero-padded column tiles
    FC_CUDA(cudaMemsetAsync(bnd, 0, 256, st));
    FC_CUDA(cudaMemsetAsync(de1, 0, static_cast<size_t>(cnt) * d * sizeof(float), st));   // reduce-add targets
    FC_CUDA(cudaMemsetAsync(de2, 0, static_cast<size_t>(cnt) * d * sizeof(float), st));
    const auto* E1 = static_cast<const __nv_bfloat16*>(e1g);
    const auto* E2 = static_cast<const __nv_bfloat16*>(e2g);
    fc::fc_rows_kernel<<<(B * 32 + 127) / 128, 128, 0, st>>>(E1, E2, B, d, lo, cnt, t1 + lo, t2 + lo, rsR, rsC, bnd,
                                                            diag);
    float* kap1 = par; float* bet1 = par + np; float* coef1 = par + 2 * np; float* fac1 = par + 3 * np;
    float* kap2 = par + 4 * np; float* bet2 = par + 5 * np; float* coef2 = par + 6 * np; float* fac2 = par + 7 * np;
    fc::fc_pair_params_kernel<<<(B + 255) / 256, 256, 0, st>>>(diag, w1, w2, t1, t2, B, kap1, bet1, coef1, fac1, kap2,
                                                               bet2, coef2, fac2, bnd);
    FC_CUDA(cudaGetLastError());
    const uint64_t rb = static_cast<uint64_t>(d) * 2;
    CUtensorMap m1k = make_map(e1g, d, B, rb, 64, 128), m2k = make_map(e2g, d, B, rb, 64, 128);
    CUtensorMap m1n = make_map(e1g, d, B, rb, 64, 64), m2n = make_map(e2g, d, B, rb, 64, 64);
    int dev = 0;
    FC_CUDA(cudaGetDevice(&dev));
    FC_CUDA(fc::sim_set_smem());   // per-device function attributes: set on the current device every call
    FC_CUDA(fc::gemm_set_smem());
    const int n_sm = sm_count(dev);
    // pass 1: row sums of S[L,G] and S^T[L,G] at the local anchors' temperatures -> r_i
    fc::SimParams sp{};
    sp.nseg = 2;
    sp.d = d;
    sp.ldq = ldq;
    sp.n_jt = n_jt;
    for (int s2 = 0; s2 < 2; ++s2) {
      fc::SimSeg& g = sp.seg[s2];
      g.rows = cnt;
      g.a_row0 = lo;
      g.cols = B;
      g.row_stat = s2 ? rsC : rsR;
      g.partial = s2 ? pC : pR;
      sp.n_rb[s2] = (cnt + fc::kPairM - 1) / fc::kPairM;
    }
    sp.n_items = (sp.n_rb[0] + sp.n_rb[1]) * n_jt;
    sp.clamps = ncl;
    sp.bounds = bnd;
    sp.n_bounds = 1;
    CUtensorMap mA[2] = {m1k, m2k}, mB[2] = {m2k, m1k};
    const int grid = 2 * std::max(1, std::min(n_sm / 2, sp.n_items));
    FC_CUDA(fc::launch_sim(fc::kSimStats, sp, mA, mB, nullptr, grid, st, nullptr));
    fc::fc_rcoef_kernel<<<(cnt + 127) / 128, 128, 0, st>>>(pR, pC, nparts, cnt, lo, w1, w2, t1, t2, rco);
    FC_CUDA(cudaGetLastError());
    // pass 2: Q'_R = Q[L,G], Q'_C = Q[G,L]^T (bf16), both from S tiles of segment R / C
    CUtensorMap mQo[2], mQ[2];
    for (int s2 = 0; s2 < 2; ++s2) {
      __nv_bfloat16* qs = q + static_cast<size_t>(s2) * cnt * ldq;
      mQo[s2] = make_map(qs, ldq, cnt, static_cast<uint64_t>(ldq) * 2, 32, 32, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                         CU_TENSOR_MAP_SWIZZLE_64B);
      mQ[s2] = make_map(qs, ldq, cnt, static_cast<uint64_t>(ldq) * 2, 64, 128);
      fc::SimSeg& g = sp.seg[s2];
      g.row_stat = nullptr;
      g.partial = nullptr;
      g.row_kappa = (s2 ? kap2 : kap1) + lo;
      g.row_beta = (s2 ? bet2 : bet1) + lo;
      g.row_coef = (s2 ? coef2 : coef1) + lo;
      g.row_fac = (s2 ? fac2 : fac1) + lo;
      g.col_kappa = s2 ? kap1 : kap2;
      g.col_beta = s2 ? bet1 : bet2;
      g.col_coef = s2 ? coef1 : coef2;
      g.col_fac = s2 ? fac1 : fac2;
      g.q = qs;
    }
    sp.q_factor = 0;   // a temperature per anchor: the two-exponential Q path
    FC_CUDA(fc::launch_sim(fc::kSimQ, sp, mA, mB, mQo, grid, st, nullptr));
    // dE = c (Q' E - r o E_L), c = 1 / (local_count (B - 1)) (engine.cpp:84-85)
    fc::GemmParams gp{};
    gp.nseg = 2;
    gp.d = d;
    gp.n_nb = (d + fc::kGemmN - 1) / fc::kGemmN;
    gp.kb_total = ldq / fc::kBlockK;
    gp.scale = static_cast<float>(1.0 / (static_cast<double>(cnt) * static_cast<double>(B - 1)));
    CUtensorMap mO[2];
    for (int s2 = 0; s2 < 2; ++s2) {
      fc::GemmSeg& g = gp.seg[s2];
      g.a_mn_major = 0;
      g.rows = cnt;
      g.x_row0 = lo;
      g.r = rco;
      g.x = s2 ? E1 : E2;
      g.out = s2 ? de2 : de1;
      gp.n_mb[s2] = (cnt + fc::kPairM - 1) / fc::kPairM;
      mO[s2] = make_map(g.out, d, cnt, static_cast<uint64_t>(d) * 4, 32, 32, CU_TENSOR_MAP_DATA_TYPE_FLOAT32);
    }
    gp.n_tiles = (gp.n_mb[0] + gp.n_mb[1]) * gp.n_nb;
    const int gemm_ctas = (n_sm / 2) * 2;
    balance_stream_k(gp, gemm_ctas / 2, 0);
    CUtensorMap mX[2] = {m2n, m1n};
    FC_CUDA(fc::launch_gemm(false, gp, mQ, mX, mO, gemm_ctas, st));
    FC_CUDA(cudaFreeAsync(ws, st));
  });
}

__global__ void fc_scale_kernel(double* x, long long n, double s) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    x[i] *= s;
}

// all_reduce_mean "grad-reduce" (trainer.cpp:540-546): sum over the ranks, then / K
// (reduce_mean, fabric.cpp:73-83; NCCL's summation order is not the fabric's ascending order).
int fc_grad_allreduce_mean(void* ctx, double* grad, int64_t n, void* stream) {
  if (!ctx || (!grad && n > 0) || n < 0) return FC_ERR_SHAPE;
  auto* s = static_cast<LossStep*>(ctx);
  return guarded([&] {
    if (s->K == 1 || n == 0) return;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    FC_NCCL(ncclAllReduce(grad, grad, static_cast<size_t>(n), ncclFloat64, ncclSum, s->comm, st));
    const long long g = std::min<long long>(4096, (n + 255) / 256);
    fc_scale_kernel<<<static_cast<int>(g), 256, 0, st>>>(grad, n, 1.0 / static_cast<double>(s->K));
    FC_CUDA(cudaGetLastError());
  });
}

int fc_comm_ledger(void* ctx, fc_ledger_entry* out, int32_t max) {
  if (!ctx || (!out && max > 0)) return -FC_ERR_SHAPE;
  auto* s = static_cast<LossStep*>(ctx);
  int n = 0;
  for (const auto& r : s->ledger) {
    if (n >= max) break;
    fc_ledger_entry& e = out[n++];
    std::memset(&e, 0, sizeof(e));
    std::strncpy(e.phase, r.phase.c_str(), sizeof(e.phase) - 1);
    e.primitive = r.primitive;
    e.world = s->K;
    e.elements = r.elements;
    e.bytes = r.bytes;
  }
  return n;
}

int fc_comm_ledger_reset(void* ctx) {
  if (!ctx) return FC_ERR_SHAPE;
  static_cast<LossStep*>(ctx)->ledger.clear();
  return FC_OK;
}

int fc_table_write(void* ctx, const char* path) {
  if (!ctx || !path) return FC_ERR_SHAPE;
  auto* s = static_cast<LossStep*>(ctx);
  return guarded([&] {
    BinOut o(path);
    write_tables(s, o);
    if (s->indiv) write_individual(s, o);
    o.check();
  });
}

int fc_table_read(void* ctx, const char* path) {
  if (!ctx || !path) return FC_ERR_SHAPE;
  auto* s = static_cast<LossStep*>(ctx);
  return guarded([&] {
    BinIn in(path);
    read_tables(s, in);
    if (s->indiv) read_individual(s, in);
  });
}

int fc_checkpoint_write(void* ctx, const char* path, const fc_model_state* model) {
  if (!ctx || !path) return FC_ERR_SHAPE;
  auto* s = static_cast<LossStep*>(ctx);
  return guarded([&] {
    fc_model_state empty{};
    const fc_model_state& m = model ? *model : empty;
    if (m.n_params < 0 || (m.n_params > 0 && (!m.params || !m.opt_m || !m.opt_v)))
      throw FcError{FC_ERR_SHAPE, "checkpoint: model arrays missing"};
    fc::TauState ts;
    FC_CUDA(cudaDeviceSynchronize());
    FC_CUDA(cudaMemcpy(&ts, s->tau_state, sizeof(ts), cudaMemcpyDeviceToHost));
    BinOut o(path);
    o.pod(kFck1Magic);
    o.pod(m.seed);
    o.pod(m.next_epoch);
    o.pod(m.global_step);
    o.raw(m.image_shape, 16);
    o.raw(m.text_shape, 16);
    std::vector<double> zero;
    o.vec(m.n_params ? m.params : zero.data(), m.n_params);
    o.vec(m.n_params ? m.opt_m : zero.data(), m.n_params);
    o.vec(m.n_params ? m.opt_v : zero.data(), m.n_params);
    o.pod(m.opt_step);
    o.pod(ts.tau);
    o.pod(ts.m);
    o.pod(ts.v);
    o.pod(ts.step);
    o.pod(static_cast<uint8_t>(ts.latched ? 1 : 0));
    write_tables(s, o);
    o.pod(static_cast<uint8_t>(s->indiv ? 1 : 0));
    if (s->indiv) write_individual(s, o);
    o.check();
  });
}

int fc_checkpoint_read(void* ctx, const char* path, fc_model_state* model) {
  if (!ctx || !path) return FC_ERR_SHAPE;
  auto* s = static_cast<LossStep*>(ctx);
  return guarded([&] {
    BinIn in(path);
    if (in.pod<uint32_t>() != kFck1Magic) throw FcError{FC_ERR_IO, std::string("bad magic in '") + path + "'"};
    fc_model_state m{};
    m.seed = in.pod<uint64_t>();
    m.next_epoch = in.pod<int64_t>();
    m.global_step = in.pod<int64_t>();
    in.raw(m.image_shape, 16);
    in.raw(m.text_shape, 16);
    const std::vector<double> params = in.vec(), om = in.vec(), ov = in.vec();
    m.n_params = static_cast<int64_t>(params.size());
    m.opt_step = in.pod<int64_t>();
    fc::TauState ts{};
    ts.tau = in.pod<double>();
    ts.m = in.pod<double>();
    ts.v = in.pod<double>();
    ts.step = in.pod<long long>();
    ts.latched = in.pod<uint8_t>() != 0;
    read_tables(s, in);
    const bool has_ind = in.pod<uint8_t>() != 0;
    if (has_ind != s->indiv)
      throw FcError{FC_ERR_CONFIG, "checkpoint: IndividualTemp presence does not match the variant"};
    if (has_ind) read_individual(s, in);
    FC_CUDA(cudaMemcpy(s->tau_state, &ts, sizeof(ts), cudaMemcpyHostToDevice));
    if (model) {
      if (model->params && model->n_params == m.n_params) {
        std::memcpy(model->params, params.data(), params.size() * 8);
        if (model->opt_m) std::memcpy(model->opt_m, om.data(), om.size() * 8);
        if (model->opt_v) std::memcpy(model->opt_v, ov.data(), ov.size() * 8);
      }
      m.params = model->params;
      m.opt_m = model->opt_m;
      m.opt_v = model->opt_v;
      *model = m;
    }
  });
}

}  // extern "C"
