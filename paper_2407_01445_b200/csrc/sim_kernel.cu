// sim_kernel.cu -- fused similarity-tile kernel (FastCLIP pass 1 and pass 2a) for sm_100a.
//
// A persistent CTA pair (cluster of 2, tcgen05 cta_group::2) walks a contiguous range of
// (segment, row block, column tile) items. Per item the pair computes one 256 x 256 tile of
// S' = A B^T (K = d) into TMEM with bf16 UMMA (M = 256 split 128/128 over the pair, N = 256
// with each CTA supplying half of B), double-buffered so the epilogue of tile t overlaps the
// MMAs of t+1. The anchor rows A stay resident in shared memory across the column tiles of a
// row block; only the contrast rows B stream (TMA ring). The epilogue never writes S:
//   STATS: per anchor row i, over the tile's columns j != i,
//            e = exp(min((s_ij - s_ii)/t_i, 60))    (safe_exp, losses.cpp:22-28)
//            sum e, sum (s_ij - s_ii) e             (engine.cpp:151-176, :182-204)
//          -> one float2 partial per (row, column quarter-tile), reduced in fixed order later.
//   Q:     Q'_ij = coef_i e_row(i,j) + coef_j e_col(i,j) (Q[i,j] = P1[i,j] + P2[j,i] of
//          engine.cpp:91-118) -> bf16 tile of the weight matrix for the gradient GEMM.
// Warp roles: w0 TMA producer, w1 MMA issuer (leader CTA), w2..w17 epilogue (4 warps per
// TMEM lane quarter, 64 columns each).
#include "kernels.cuh"
#include "sm100.cuh"

namespace fc {

// cycle counters / globaltimer stamps into SimParams::dbg_out: profiling builds only
// (FC_PROFILE=1 python -m paper_2407_01445_b200.build); the shipped library compiles them out
#ifdef FC_PROFILE
constexpr bool kProf = true;
#else
constexpr bool kProf = false;
#endif

namespace {

constexpr float kClampLog2 = 60.0f * 1.4426950408889634f;  // kExpClampMax in the log2 domain

struct SmemLayout {
  uint8_t* a;          // kSimASlots x 16 KB: resident anchor rows (one K block per slot)
  uint8_t* b;          // kStagesB x 16 KB: streamed contrast rows
  float* par;          // kSimPSlots x {kappa[256], beta[256], coef[256], fac[256]} (Q pass)
  uint8_t* qout;       // kSimEpiWarps x 2 KB: Q store staging (Q pass)
  uint64_t* full;      // B ring
  uint64_t* empty;
  uint64_t* afull;     // A slots
  uint64_t* aempty;
  uint64_t* tfull;     // TMEM accumulators
  uint64_t* tempty;
  uint64_t* pfull;     // column-parameter slots
  uint64_t* pempty;
  uint32_t* tmem_ptr;
};

template <int kStagesB>
__device__ __forceinline__ SmemLayout carve(uint8_t* base) {
  SmemLayout L;
  uint8_t* p = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(base) + 1023) & ~uintptr_t(1023));
  L.a = p;
  L.b = p + kSimASlots * kStageBytesA;
  L.qout = L.b + kStagesB * kStageBytesB;
  L.par = reinterpret_cast<float*>(L.qout + (kStagesB == kSimStagesQ ? kSimEpiWarps * kSimStageOutQ : 0));
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(L.par) +
                                               (kStagesB == kSimStagesQ ? kSimPSlots * kSimPSlotBytes : kSimParRedBytes));
  L.full = bars;
  L.empty = L.full + kStagesB;
  L.afull = L.empty + kStagesB;
  L.aempty = L.afull + kSimASlots;
  L.tfull = L.aempty + kSimASlots;
  L.tempty = L.tfull + 2;
  L.pfull = L.tempty + 2;
  L.pempty = L.pfull + kSimPSlots;
  L.tmem_ptr = reinterpret_cast<uint32_t*>(L.pempty + kSimPSlots);
  return L;
}

// Work of one pair: q = floor(T / P) whole 256x256 tiles, contiguous (the resident anchor rows
// A carry over between them), then the R = T mod P leftover tiles split into 2R half tiles
// (256 x 128, UMMA N = 128) dealt round-robin, so the slowest pair runs q + 1/2 tiles
// instead of q + 1.
struct PairItems {
  int q, tail_lo, n_pairs, pair, count;
  int n_own, rem_lo;   // local-first order: own-tile items, first remote item
};
template <bool kLF>
__device__ __forceinline__ PairItems pair_items(const SimParams& p, int n_tiles, int pair, int n_pairs, bool split) {
  PairItems pi;
  pi.n_pairs = n_pairs;
  pi.pair = pair;
  if (kLF && p.local_first) {
    // two lists in group order -- every (segment, row block) group's own tiles, then every
    // group's remote tiles. The pair takes a contiguous share of each: the same fraction of the
    // own list, and of the remote list what makes its total the balanced share of all tiles
    // (floor(T (p+1) / P) - floor(T p / P); the host launches at most T / 2 pairs, which keeps
    // the remote shares non-negative). Both shares cover about the same groups, so A mostly
    // stays resident; the remote share runs in reverse, starting in the group the own share ended in.
    const long long n_grp = n_tiles / p.n_jt;
    const long long own = n_grp * p.n_loc;
    const int c_lo = static_cast<int>(static_cast<long long>(n_tiles) * pair / n_pairs);
    const int c_hi = static_cast<int>(static_cast<long long>(n_tiles) * (pair + 1) / n_pairs);
    pi.q = -2;
    pi.tail_lo = static_cast<int>(own * pair / n_pairs);
    pi.n_own = static_cast<int>(own * (pair + 1) / n_pairs) - pi.tail_lo;
    pi.rem_lo = c_lo - pi.tail_lo;
    pi.count = max(c_hi - c_lo, pi.n_own);
    return pi;
  }
  if (!split) {   // contiguous ranges of whole tiles
    pi.q = -1;
    pi.tail_lo = static_cast<int>((static_cast<long long>(n_tiles) * pair) / n_pairs);
    pi.count = static_cast<int>((static_cast<long long>(n_tiles) * (pair + 1)) / n_pairs) - pi.tail_lo;
    return pi;
  }
  pi.q = n_tiles / n_pairs;
  pi.tail_lo = pi.q * n_pairs;   // first leftover tile
  const int halves = 2 * (n_tiles - pi.tail_lo);
  pi.count = pi.q + (pair < halves ? (halves - pair + n_pairs - 1) / n_pairs : 0);
  return pi;
}
// item -> (segment, row block, column tile, half: -1 whole tile, 0 / 1 the column half)
template <bool kLF>
__device__ __forceinline__ void decode_item(const SimParams& p, const PairItems& pi, int item, int& s, int& rb,
                                            int& jt, int& half) {
  int t;
  if (kLF && pi.q == -2) {   // local-first order
    int grp;
    if (item < pi.n_own) {
      const int u = pi.tail_lo + item;
      grp = u / p.n_loc;
      jt = p.jt_lo + u % p.n_loc;
    } else {
      const int n_rem = p.n_jt - p.n_loc;
      const int v = pi.rem_lo + (pi.count - 1 - item);   // reverse order
      grp = v / n_rem;
      const int r = v % n_rem;
      jt = r < p.jt_lo ? r : r + p.n_loc;
    }
    half = -1;
    s = grp < p.n_rb[0] ? 0 : 1;
    rb = grp - (s ? p.n_rb[0] : 0);
    return;
  }
  if (pi.q < 0) {
    t = pi.tail_lo + item;
    half = -1;
  } else if (item < pi.q) {
    t = pi.pair * pi.q + item;
    half = -1;
  } else {
    const int h = pi.pair + (item - pi.q) * pi.n_pairs;
    t = pi.tail_lo + h / 2;
    half = h & 1;
  }
  const int n0 = p.n_rb[0] * p.n_jt;
  s = t < n0 ? 0 : 1;
  const int local = t - (s ? n0 : 0);
  rb = local / p.n_jt;
  jt = local % p.n_jt;
}
// Identity of the A block an (item, chunk) needs: segment, row block, 512-wide K chunk.
template <bool kLF>
__device__ __forceinline__ int a_key(const SimParams& p, const PairItems& pi, int item, int chunk, int n_chunks) {
  int s, rb, jt, half;
  decode_item<kLF>(p, pi, item, s, rb, jt, half);
  return ((s * 65536) + rb) * n_chunks + chunk;
}

// Inserts `id` into the step's id set; false when it is already there. Slots hold
// (tag << 32) | id with tag = low 32 bits of the step sequence number + 1: slots of earlier
// steps read as free.
__device__ bool idset_insert(unsigned long long* set, int mask, unsigned long long seq, int id) {
  const unsigned long long tag = ((seq & 0xffffffffull) + 1ull) << 32;
  const unsigned long long key = tag | static_cast<unsigned int>(id);
  unsigned int h = (static_cast<unsigned int>(id) * 2654435761u) & static_cast<unsigned int>(mask);
  for (;;) {
    unsigned long long v = set[h];
    while ((v & 0xffffffff00000000ull) != tag) {   // stale slot: claim it
      const unsigned long long old = atomicCAS(set + h, v, key);
      if (old == v) return true;
      v = old;
    }
    if (v == key) return false;
    h = (h + 1) & static_cast<unsigned int>(mask);
  }
}

__device__ __forceinline__ void bulk_load(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(smem)),
      "l"(reinterpret_cast<uint64_t>(gmem)), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ---- epilogue chunk processors (32 consecutive columns of one row per thread) ----
// Exponents are formed directly in the log2 domain with one FMA, y = s*kappa + beta where
// kappa = log2(e)/t and beta = -S_aa*kappa, and the packed fp32x2 pipe (FFMA2/FADD2) does
// two elements per instruction. The fast paths skip the safe_exp clamp and the masks; a
// warp-uniform check of the chunk's max exponent routes the (rare) clamped chunks, and the
// ragged/diagonal chunks, to the exact slow path.
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

// STATS fast path: chunk sums of e and y*e (sum (s - S_ii) e = sum(y e) / kappa).
__device__ __forceinline__ void stats_fast(const uint32_t (&r)[32], float kap, float beta, float2& se, float2& sye) {
  const float2 k2 = f2(kap, kap), b2 = f2(beta, beta);
#pragma unroll
  for (int k = 0; k < 32; k += 2) {
    const float2 y = __ffma2_rn(f2(__uint_as_float(r[k]), __uint_as_float(r[k + 1])), k2, b2);
    const float2 e = f2(ex2_approx(y.x), ex2_approx(y.y));
    se = __fadd2_rn(se, e);
    sye = __ffma2_rn(y, e, sye);
  }
}
// STATS exact path: clamp (safe_exp), masks, clamp count.
__device__ __forceinline__ void stats_masked(const uint32_t (&r)[32], float kap, float beta, int col0, int cols, int gi,
                                             bool row_ok, float& se, float& sye, uint32_t& ncl) {
#pragma unroll
  for (int k = 0; k < 32; ++k) {
    const int j = col0 + k;
    const float y = fmaf(__uint_as_float(r[k]), kap, beta);
    const bool ok = row_ok && (j < cols) && (j != gi);
    const float e = ex2_approx(fminf(y, kClampLog2));
    se += ok ? e : 0.f;
    sye += ok ? y * e : 0.f;
    ncl += (ok && y > kClampLog2) ? 1u : 0u;
  }
}

// Column sums of a warp's 32-row x N-column piece (N = 32 or 8): lane l holds row l's N
// values; the rows are folded pairwise (xor 16 .. N), then log2(N) xor-halving steps leave the
// sum of column (l % N) in lane l (31 shuffles per array for N = 32).
template <int N>
__device__ __forceinline__ float transpose_reduce(float (&v)[N], uint32_t lane) {
#pragma unroll
  for (int w = 16; w >= N; w >>= 1)
#pragma unroll
    for (int k = 0; k < N; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k], w);
#pragma unroll
  for (int w = N / 2; w >= 1; w >>= 1) {
    const bool upper = (lane & w) != 0;
#pragma unroll
    for (int k = 0; k < w; ++k) {
      const float send = upper ? v[k] : v[k + w];
      const float keep = upper ? v[k + w] : v[k];
      v[k] = keep + __shfl_xor_sync(0xffffffffu, send, w);
    }
  }
  return v[0];
}

// Column sums of two 32 x 16 register tiles in lock-step (lane = row): the xor-halving over
// lane bits 3..0 leaves column (lane & 15)'s sum over the 16 rows of the lane's half-warp, one
// more xor-16 step adds the other half (both lanes of a pair then hold the full column sum).
__device__ __forceinline__ void transpose_reduce2_16(float (&v)[16], float (&u)[16], uint32_t lane, float& sv,
                                                     float& su) {
#pragma unroll
  for (int w = 8; w >= 1; w >>= 1) {
    const bool upper = (lane & w) != 0;
#pragma unroll
    for (int k = 0; k < w; ++k) {
      const float sv_ = upper ? v[k] : v[k + w];
      const float kv = upper ? v[k + w] : v[k];
      const float su_ = upper ? u[k] : u[k + w];
      const float ku = upper ? u[k + w] : u[k];
      v[k] = kv + __shfl_xor_sync(0xffffffffu, sv_, w);
      u[k] = ku + __shfl_xor_sync(0xffffffffu, su_, w);
    }
  }
  sv = v[0] + __shfl_xor_sync(0xffffffffu, v[0], 16);
  su = u[0] + __shfl_xor_sync(0xffffffffu, u[0], 16);
}

// FUSED fast path (one temperature, no clamp possible, no diagonal / ragged element in the
// chunk): x = 2^(s kappa) once per element serves the row (R) and the column (C) statistics,
// e_row = 2^beta_i x, e_col = 2^beta_j x. Row raw sums {sum x, sum z x} (z = s kappa)
// accumulate per thread; lane c (c < 16) or c + 16 (c >= 16) gets that column's raw sums of the 16-column half.
__device__ __forceinline__ void fused_fast16(const uint32_t (&r)[16], float kap, float2& rx, float2& rzx, uint32_t lane,
                                             float& cx, float& czx) {
  const float2 k2 = f2(kap, kap);
  float x[16], zx[16];
#pragma unroll
  for (int k = 0; k < 16; k += 2) {
    const float2 z = __fmul2_rn(f2(__uint_as_float(r[k]), __uint_as_float(r[k + 1])), k2);
    const float2 e = f2(ex2_approx(z.x), ex2_approx(z.y));
    const float2 ze = __fmul2_rn(z, e);
    rx = __fadd2_rn(rx, e);
    rzx = __fadd2_rn(rzx, ze);
    x[k] = e.x; x[k + 1] = e.y;
    zx[k] = ze.x; zx[k + 1] = ze.y;
  }
  transpose_reduce2_16(x, zx, lane, cx, czx);
}

// FUSED clamp-free two-exponential path (no clamp possible in the chunk, no diagonal / ragged
// element, but outside the one-exponential form: a temperature per anchor (v2 / iSogCLR) or
// kappa |s| > 63 (tau below ~0.023)): e_row = 2^(s kappa_i + beta_i) and e_col = 2^(s kappa_j +
// beta_j) per element, the column anchors' {kappa_j, beta_j} broadcast from the lanes holding them
// (one shuffle per column and warp, not per element). Row sums {sum e, sum y e} accumulate per
// thread; the column sums go through the same register transposes as the one-exponential path.
template <bool kOneKappa>
__device__ __forceinline__ void fused_2e16(const uint32_t (&r)[16], float2 rs, float2 cs, int c0, uint32_t lane,
                                           float2& re, float2& rye, float& ce, float& cye) {
  const float2 rk2 = f2(rs.x, rs.x), rb2 = f2(rs.y, rs.y);
  float x[16], zx[16];
#pragma unroll
  for (int k = 0; k < 16; k += 2) {
    const float2 s = f2(__uint_as_float(r[k]), __uint_as_float(r[k + 1]));
    const float2 yr = __ffma2_rn(s, rk2, rb2);
    const float b0 = __shfl_sync(0xffffffffu, cs.y, c0 + k), b1 = __shfl_sync(0xffffffffu, cs.y, c0 + k + 1);
    float2 kc = rk2;
    if constexpr (!kOneKappa)
      kc = f2(__shfl_sync(0xffffffffu, cs.x, c0 + k), __shfl_sync(0xffffffffu, cs.x, c0 + k + 1));
    const float2 yc = __ffma2_rn(s, kc, f2(b0, b1));
    const float2 er = f2(ex2_approx(yr.x), ex2_approx(yr.y));
    const float2 ec = f2(ex2_approx(yc.x), ex2_approx(yc.y));
    re = __fadd2_rn(re, er);
    rye = __ffma2_rn(yr, er, rye);
    const float2 ze = __fmul2_rn(yc, ec);
    x[k] = ec.x; x[k + 1] = ec.y;
    zx[k] = ze.x; zx[k + 1] = ze.y;
  }
  transpose_reduce2_16(x, zx, lane, ce, cye);
}

// FUSED exact path for one 8-column piece (rare: diagonal / ragged / clamp-capable chunks):
// both exponentials with the safe_exp clamp, masks and clamp counts; the lanes of quarter q of
// the warp get their column's exact {sum e, sum y e}.
__device__ __forceinline__ void fused_masked(const uint32_t (&r)[8], float2 rs, const float2* __restrict__ cs, int c0,
                                             int cols, int gi, bool row_ok, uint32_t lane, int q, float& se,
                                             float& sye, uint32_t& ncl, float& ce, float& cye) {
  float x[8], yx[8];
  // lane l loads column (c0 + l % 8)'s parameters once; element k reads them by shuffle
  const int jl = c0 + static_cast<int>(lane & 7);
  const float2 cl = jl < cols ? cs[jl] : f2(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const int j = c0 + k;
    const bool ok = row_ok && (j < cols) && (j != gi);
    const float s = __uint_as_float(r[k]);
    const float yr = fmaf(s, rs.x, rs.y);
    const float yc = fmaf(s, __shfl_sync(0xffffffffu, cl.x, k), __shfl_sync(0xffffffffu, cl.y, k));
    const float er = ex2_approx(fminf(yr, kClampLog2));
    const float ec = ex2_approx(fminf(yc, kClampLog2));
    se += ok ? er : 0.f;
    sye += ok ? yr * er : 0.f;
    ncl += (ok && yr > kClampLog2) ? 1u : 0u;
    ncl += (ok && yc > kClampLog2) ? 1u : 0u;
    x[k] = ok ? ec : 0.f;
    yx[k] = ok ? yc * ec : 0.f;
  }
  const float a = transpose_reduce<8>(x, lane);
  const float b = transpose_reduce<8>(yx, lane);
  if ((lane >> 3) == static_cast<uint32_t>(q)) { ce = a; cye = b; }
}

// Q with one temperature for every anchor (kappa_i = kappa_j): the two exponentials share
// 2^(s kappa), so Q'_ij = 2^(s kappa) (fac_i + fac_j) with fac_a = coef_a 2^beta_a -- one
// MUFU ex2 per element instead of two (pass 2 is otherwise SFU-bound at the MMA rate).
constexpr float kFactMaxLog2 = 63.0f;
__device__ __forceinline__ void q_chunk_fact(const uint32_t (&r)[32], float rk, float rf, const float* fc,
                                             uint32_t (&packed)[16]) {
  const float2 rk2 = f2(rk, rk), rf2 = f2(rf, rf);
#pragma unroll
  for (int k = 0; k < 32; k += 4) {
    const float4 ff = *reinterpret_cast<const float4*>(fc + k);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float2 s = f2(__uint_as_float(r[k + 2 * h]), __uint_as_float(r[k + 2 * h + 1]));
      const float2 y = __fmul2_rn(s, rk2);
      const float2 e = f2(ex2_approx(y.x), ex2_approx(y.y));
      const float2 q = __fmul2_rn(e, __fadd2_rn(rf2, h ? f2(ff.z, ff.w) : f2(ff.x, ff.y)));
      __nv_bfloat162 hq = __floats2bfloat162_rn(q.x, q.y);
      packed[k / 2 + h] = *reinterpret_cast<uint32_t*>(&hq);
    }
  }
}

// Q: 32 bf16 weights of one row; col params from shared memory (broadcast reads).
template <bool kExact>
__device__ __forceinline__ void q_chunk(const uint32_t (&r)[32], float rk, float rb, float rc, const float* kc,
                                         const float* bc, const float* cc, int col0, int cols, int gi,
                                         uint32_t (&packed)[16]) {
  const float2 rk2 = f2(rk, rk), rb2 = f2(rb, rb), rc2 = f2(rc, rc);
#pragma unroll
  for (int k = 0; k < 32; k += 4) {
    const float4 kk = *reinterpret_cast<const float4*>(kc + k);
    const float4 bb = *reinterpret_cast<const float4*>(bc + k);
    const float4 cf = *reinterpret_cast<const float4*>(cc + k);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float2 s = f2(__uint_as_float(r[k + 2 * h]), __uint_as_float(r[k + 2 * h + 1]));
      const float2 kc2 = h ? f2(kk.z, kk.w) : f2(kk.x, kk.y);
      const float2 bc2 = h ? f2(bb.z, bb.w) : f2(bb.x, bb.y);
      const float2 cc2 = h ? f2(cf.z, cf.w) : f2(cf.x, cf.y);
      float2 yr = __ffma2_rn(s, rk2, rb2);
      float2 yc = __ffma2_rn(s, kc2, bc2);
      if constexpr (kExact) {
        yr = f2(fminf(yr.x, kClampLog2), fminf(yr.y, kClampLog2));
        yc = f2(fminf(yc.x, kClampLog2), fminf(yc.y, kClampLog2));
      }
      const float2 er = f2(ex2_approx(yr.x), ex2_approx(yr.y));
      const float2 ec = f2(ex2_approx(yc.x), ex2_approx(yc.y));
      float2 q = __ffma2_rn(cc2, ec, __fmul2_rn(rc2, er));
      if constexpr (kExact) {
        const int j = col0 + k + 2 * h;
        q.x = (j < cols && j != gi) ? q.x : 0.f;
        q.y = (j + 1 < cols && j + 1 != gi) ? q.y : 0.f;
      }
      __nv_bfloat162 hq = __floats2bfloat162_rn(q.x, q.y);
      packed[k / 2 + h] = *reinterpret_cast<uint32_t*>(&hq);
    }
  }
}

}  // namespace

// Epilogue shape (every mode): 16 epilogue warps, 4 per TMEM lane quarter, 64 columns each; the
// FUSED path works in 16-column halves so its transposes fit the 96-register budget.
template <int kMode>
struct SimCfg {
  static constexpr int kEpi = kSimEpiWarps;
  static constexpr int kThreads = (kEpi + 2) * 32;
  static constexpr int kColsW = kPairN / (kEpi / 4);   // columns per epilogue warp
  static constexpr int kChunksW = kColsW / 32;
};

template <int kMode>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(SimCfg<kMode>::kThreads, 1)
    sim_tile_kernel(const __grid_constant__ SimParams p, const __grid_constant__ CUtensorMap mapA0,
                    const __grid_constant__ CUtensorMap mapB0, const __grid_constant__ CUtensorMap mapA1,
                    const __grid_constant__ CUtensorMap mapB1, const __grid_constant__ CUtensorMap mapQo0,
                    const __grid_constant__ CUtensorMap mapQo1, float* __restrict__ raw_out) {
  constexpr int kStagesB = kMode == kSimQ ? kSimStagesQ : kSimStagesStats;
  constexpr bool kLF = kMode == kSimStats || kMode == kSimQ;   // the passes that run beside a gather (K > 1)
  constexpr bool kStatsLike = kMode == kSimStats || kMode == kSimFused;
  extern __shared__ uint8_t smem_raw[];
  long long g_entry = 0;
  if (kProf) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_entry));
  const SmemLayout L = carve<kStagesB>(smem_raw);
  const uint32_t warp = threadIdx.x / 32;
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x / 2;
  const int n_pairs = gridDim.x / 2;
  const int nkb = (p.d + kBlockK - 1) / kBlockK;

  // warp roles: epilogue warps first, producer and MMA issuer LAST -- the SMSP arbiter
  // favours the highest warp id, so the single-thread TMA/MMA issue never waits behind
  // the epilogue math.
  constexpr int kEpi = SimCfg<kMode>::kEpi;
  constexpr int kColsW = SimCfg<kMode>::kColsW;
  constexpr int kChunksW = SimCfg<kMode>::kChunksW;
  constexpr uint32_t kProdWarp = kEpi, kMmaWarp = kEpi + 1;
  if (warp == kProdWarp && lane == 0) {
    tma_prefetch(&mapA0);
    tma_prefetch(&mapB0);
    if (p.nseg > 1) {
      tma_prefetch(&mapA1);
      tma_prefetch(&mapB1);
    }
  }
  if (warp == kMmaWarp && lane == 0) {
    for (int i = 0; i < kStagesB; ++i) {
      mbar_init(&L.full[i], 2);   // leader's expect_tx arrive + peer's remote arrive
      mbar_init(&L.empty[i], 1);  // MMA commit (multicast to both CTAs)
    }
    for (int i = 0; i < kSimASlots; ++i) {
      mbar_init(&L.afull[i], 2);
      mbar_init(&L.aempty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&L.tfull[i], 1);                    // MMA commit (multicast)
      mbar_init(&L.tempty[i], 2 * kEpi);            // one arrive per epilogue warp of the pair
    }
    for (int i = 0; i < kSimPSlots; ++i) {
      mbar_init(&L.pfull[i], 1);                    // local producer + bulk-copy bytes
      mbar_init(&L.pempty[i], kEpi);                // local epilogue warps

    }
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<2>(L.tmem_ptr, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *L.tmem_ptr;
  // the next kernel may take SMs as this grid's CTAs retire. Local-first: only once the producer
  // saw every gather flag -- the dependent grid's early CTAs would otherwise take the room a
  // gather CTA needs beside this one (this grid waits for that gather)
  if (!p.local_first) griddep_launch_dependents();

  const int n_chunks = (nkb + kSimASlots - 1) / kSimASlots;
  const PairItems pi = pair_items<kLF>(p, p.n_items, pair, n_pairs, p.split_tail != 0);
  const int it_lo = 0, it_hi = pi.count;

  if (warp == kProdWarp) {
    // ===================== TMA producer (both CTAs) =====================
    // A (anchor rows, own 128 of the pair's 256) is loaded once per (segment, row block,
    // K chunk) into per-K-block slots; each slot is refilled as soon as the MMAs of the last
    // tile that read it retire (aempty), so the switch to the next row block overlaps.
    // The whole warp walks the loop (warp-uniform waits); lane 0 issues. A single-thread loop
    // in a diverged warp wakes from mbarrier waits noticeably later.
    {
      const bool issuer = lane == 0;
      uint32_t stage = 0, phase = 0;
      uint32_t spar = 0;   // bit per A slot: parity of its load generation (afull/aempty phase), kept in a register
      int cur_key = -1;
      int it = 0;
      // local-first (K > 1): what rank k's gather writes (pass 1: its rows of the gathered
      // embeddings; pass 2: its anchors' column parameters) is read only after rank k's flag
      // carries this step's sequence number (set by the gather kernel running beside this grid)
      uint32_t seen = 0;
      unsigned long long seq = 0;
      auto wait_rank = [&](int k) {
        if ((seen >> k) & 1u) return;
        if (seen == 0) {
          griddep_wait();   // the step tag is written by the preceding kernel
          seq = *p.step_tag;
        }
        if (issuer) {
          unsigned spins = 0;
          long long t0 = 0;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
          while (ld_relaxed_sys(p.src_flag + k) < seq) {
            __nanosleep(32);
            if ((++spins & 255u) != 0u) continue;
            // a poisoned collective (the gather kernel's timeout), or no flag within the peer
            // timeout (e.g. the gather never got an SM): stop waiting, report it
            long long t1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            if (ld_relaxed_sys(p.abort_flag) != 0ull || t1 - t0 > p.timeout_ns) {
              atomicCAS(p.err, 0, 8 /* FC_ERR_COLLECTIVE_ABORTED */);
              break;
            }
          }
          // acquire through the flag (an acquire load, not a fence.sys: that would drain this SM's
          // outstanding traffic), then order the peer's rows for the TMA (async-proxy) reads
          (void)ld_acquire_sys(p.src_flag + k);
          fence_proxy_async_global();
        }
        __syncwarp();
        seen |= 1u << k;
      };
      // column parameters of the pair's j-th tile (each CTA keeps its own copy), written by the
      // preceding per-anchor kernel: the first load waits for that grid (programmatic launch;
      // the A / B operand loads do not depend on it)
      // columns [jt * 256, +256) of a tile: wait for every rank that holds some of them
      auto wait_tile = [&](int s, int jt) {
        const int c_hi = min(jt * kPairN + kPairN, p.seg[s].cols) - 1;
        for (int k = (jt * kPairN) / p.rows_per_src; k <= c_hi / p.rows_per_src; ++k) wait_rank(k);
      };
      auto load_params = [&](int j) {
        int s, rb, jt, half;
        decode_item<kLF>(p, pi, it_lo + j, s, rb, jt, half);
        if (j == 0) griddep_wait();
        if (p.local_first == 2 && !(jt >= p.jt_lo && jt < p.jt_lo + p.n_loc)) wait_tile(s, jt);
        const int ps = j % kSimPSlots;
        mbar_wait(&L.pempty[ps], ((j / kSimPSlots) & 1) ^ 1);
        if (issuer) {
          mbar_arrive_expect_tx(&L.pfull[ps], kSimPSlotBytes);
          float* dst = L.par + ps * (kSimPSlotBytes / 4);
          const SimSeg& sg = p.seg[s];
          bulk_load(dst, sg.col_kappa + jt * kPairN, kPairN * 4, &L.pfull[ps]);
          bulk_load(dst + kPairN, sg.col_beta + jt * kPairN, kPairN * 4, &L.pfull[ps]);
          bulk_load(dst + 2 * kPairN, sg.col_coef + jt * kPairN, kPairN * 4, &L.pfull[ps]);
          bulk_load(dst + 3 * kPairN, sg.col_fac + jt * kPairN, kPairN * 4, &L.pfull[ps]);
        }
        __syncwarp();
      };
      for (int item = it_lo; item < it_hi; ++item, ++it) {
        int s, rb, jt, half;
        decode_item<kLF>(p, pi, item, s, rb, jt, half);
        // pass 1 (local_first 1): own tiles and A from the caller's slices
        const bool own = p.local_first == 1 && jt >= p.jt_lo && jt < p.jt_lo + p.n_loc;
        const CUtensorMap* ma = s ? &mapA1 : &mapA0;
        const CUtensorMap* mb = own ? (s ? &mapQo1 : &mapQo0) : (s ? &mapB1 : &mapB0);
        const int a_row = p.seg[s].a_row0 - (p.local_first == 1 ? p.col_lo : 0) + rb * kPairM + static_cast<int>(rank) * kCtaM;
        // each CTA supplies half of the tile's columns: 128 of a whole tile, 64 of a half tile
        // (the 128-row box then also brings 64 rows the UMMA does not read)
        const int b_row = (half < 0 ? jt * kPairN + static_cast<int>(rank) * (kPairN / 2)
                                    : jt * kPairN + half * (kPairN / 2) + static_cast<int>(rank) * (kPairN / 4)) -
                          (own ? p.col_lo : 0);
        if (p.local_first == 1 && !own) wait_tile(s, jt);
        // params ahead of the tile's operands, except for the pair's first tile: its operands
        // go out first, so its MMAs run while the per-anchor kernel is still producing the
        // parameters (the first param load is the grid-dependency wait)
        if constexpr (kMode == kSimQ) if (it >= 1) load_params(it);
        for (int c = 0; c < n_chunks; ++c) {
          const int kb_lo = c * kSimASlots;
          const int kb_hi = min(nkb, kb_lo + kSimASlots);
          const int key = a_key<kLF>(p, pi, item, c, n_chunks);
          const bool new_a = key != cur_key;
          cur_key = key;
          // a new A block goes out k block by k block, each A slot right before the B stage of
          // the same k block (the first MMA needs 32 KB per CTA, not the whole 128 KB of A)
          for (int kb = kb_lo; kb < kb_hi; ++kb) {
            if (new_a) {
              const int slot = kb - kb_lo;
              mbar_wait(&L.aempty[slot], ((spar >> slot) & 1) ^ 1);
              spar ^= 1u << slot;
              if (issuer) {
                if (rank == 0) mbar_arrive_expect_tx(&L.afull[slot], 2 * kStageBytesA);
                else mbar_arrive_cluster(&L.afull[slot], 0);
                tma_load_2d_pair(ma, &L.afull[slot], L.a + slot * kStageBytesA, kb * kBlockK, a_row);
              }
              __syncwarp();
            }
            mbar_wait(&L.empty[stage], phase ^ 1);
            if (issuer) {
              if (rank == 0) mbar_arrive_expect_tx(&L.full[stage], 2 * kStageBytesB);
              else mbar_arrive_cluster(&L.full[stage], 0);
              tma_load_2d_pair(mb, &L.full[stage], L.b + stage * kStageBytesB, kb * kBlockK, b_row);
            }
            __syncwarp();
            if (++stage == kStagesB) { stage = 0; phase ^= 1; }
          }
        }
        if constexpr (kMode == kSimQ) if (it == 0) load_params(0);
      }
      // the later kernels of the step read the whole gathered buffers: every rank's flag (this
      // rank's own gather included) is observed before this grid completes (pass 1). For
      // pass 2: this rank's own gather included, so the step's later bounds reset cannot
      // precede any of the payload gather's stores
      if (p.local_first) {
        for (int k = 0; k * p.rows_per_src < p.seg[0].cols; ++k) wait_rank(k);
        griddep_launch_dependents();
      }
    }
  } else if (warp == kMmaWarp) {
    // ===================== MMA issuer (leader CTA only, one thread) =====================
    // The issue loop is kept lean (precomputed descriptors, no per-MMA address math, no
    // warp-wide election per k block): with ~100+ cycles of scalar work per MMA the single
    // issuing thread, not the tensor pipe, would set the pace (128 cycles per 256x256x16).
    if (rank == 0) {
      constexpr uint32_t idesc_full = make_idesc_bf16(kPairM, kPairN, 0, 0);
      constexpr uint32_t idesc_half = make_idesc_bf16(kPairM, kPairN / 2, 0, 0);
      const uint64_t a_desc0 = make_sdesc_sw128(smem_u32(L.a), 0, 1024);
      const uint64_t b_desc0 = make_sdesc_sw128(smem_u32(L.b), 0, 1024);
      uint32_t stage = 0, phase = 0;
      uint32_t spar = 0;   // bit per A slot: parity of the generation being consumed + 1
      uint32_t ready = 0;   // bit per A slot: afull of the current generation observed
      int cur_key = -1;
      int it = 0;
      constexpr bool prof = kProf;
      long long c_start = clock64(), c_tempty = 0, c_afull = 0, c_full = 0, c_first = 0, n_mma = 0;
      for (int item = it_lo; item < it_hi; ++item, ++it) {
        const uint32_t acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        long long t0 = prof ? clock64() : 0;
        mbar_wait(&L.tempty[acc], acc_phase ^ 1);
        if (prof) c_tempty += clock64() - t0;
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kPairN;
        int s_, rb_, jt_, half_;
        decode_item<kLF>(p, pi, item, s_, rb_, jt_, half_);
        const uint32_t idesc = half_ < 0 ? idesc_full : idesc_half;
        for (int c = 0; c < n_chunks; ++c) {
          const int kb_lo = c * kSimASlots;
          const int kb_hi = min(nkb, kb_lo + kSimASlots);
          const int key = a_key<kLF>(p, pi, item, c, n_chunks);
          if (key != cur_key) {
            cur_key = key;
            ready = 0;
            spar ^= (1u << (kb_hi - kb_lo)) - 1u;
          }
          // last use of this A generation: release each slot right after its MMAs
          int nxt_key = -2;
          if (c + 1 < n_chunks) nxt_key = a_key<kLF>(p, pi, item, c + 1, n_chunks);
          else if (item + 1 < it_hi) nxt_key = a_key<kLF>(p, pi, item + 1, 0, n_chunks);
          const bool last_use = nxt_key != key;
          const bool last_chunk = c == n_chunks - 1;
          for (int kb = kb_lo; kb < kb_hi; ++kb) {
            const int slot = kb - kb_lo;
            if (!(ready & (1u << slot))) {
              long long t1 = prof ? clock64() : 0;
              mbar_wait(&L.afull[slot], ((spar >> slot) & 1) ^ 1);
              if (prof) c_afull += clock64() - t1;
              ready |= 1u << slot;
            }
            long long t2 = prof ? clock64() : 0;
            mbar_wait(&L.full[stage], phase);
            if (prof) {
              c_full += clock64() - t2;
              if (n_mma == 0) c_first = clock64() - c_start;
              n_mma += 4;
            }
            tc_fence_after();
            if (elect_one()) {
              const uint64_t ad = a_desc0 + static_cast<uint64_t>((slot * kStageBytesA) >> 4);
              const uint64_t bd = b_desc0 + static_cast<uint64_t>((stage * kStageBytesB) >> 4);
              mma_bf16_pair(d_tmem, ad, bd, idesc, kb != 0);
              mma_bf16_pair(d_tmem, ad + 2, bd + 2, idesc, 1);
              mma_bf16_pair(d_tmem, ad + 4, bd + 4, idesc, 1);
              mma_bf16_pair(d_tmem, ad + 6, bd + 6, idesc, 1);
              mma_commit_pair(&L.empty[stage], 0x3);
              if (last_use) mma_commit_pair(&L.aempty[slot], 0x3);
              if (last_chunk && kb == kb_hi - 1) mma_commit_pair(&L.tfull[acc], 0x3);
            }
            __syncwarp();
            if (++stage == kStagesB) { stage = 0; phase ^= 1; }
          }
        }
      }
      if (prof && lane == 0) {
        long long* o = p.dbg_out + pair * 8;
        o[0] = clock64() - c_start; o[1] = c_tempty; o[2] = c_afull; o[3] = c_full; o[4] = c_first; o[5] = n_mma;
        o[6] = it_hi - it_lo;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(o[7]));   // MMA loop end (ns)
      }
    }
  } else {
    // ===================== epilogue (both CTAs) =====================
    if (p.zero_n4 > 0) {   // dE <- 0 (nothing of this step reads it before the GEMM)
      const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
      const long long nt = static_cast<long long>(gridDim.x) * kEpi * 32;
      for (long long g = static_cast<long long>(blockIdx.x) * kEpi * 32 + threadIdx.x; g < p.zero_n4; g += nt) {
        p.zero0[g] = z;
        p.zero1[g] = z;
      }
    }
    griddep_wait();   // row / column parameters and bounds come from the preceding kernel
    if (p.idset) {
      // duplicate-id check: every epilogue thread of the grid inserts at most a few of the rank's
      // ids (one L2 round trip before its first accumulator wait, overlapping the first MMAs)
      const unsigned long long seq = *p.step_tag;   // written by prep (this grid's predecessor)
      bool dup = false;
      for (int i = blockIdx.x * kEpi * 32 + static_cast<int>(threadIdx.x); i < p.n_ids; i += gridDim.x * kEpi * 32) {
        const int id = p.ids[i];
        if (id >= 0 && !idset_insert(p.idset, p.idset_mask, seq, id)) dup = true;
      }
      // a repeated id: the reference's owner check (state.cpp:47-49) rejects the write
      if (__any_sync(0xffffffffu, dup) && lane == 0) atomicCAS(p.err, 0, 5 /* FC_ERR_OWNERSHIP */);
    }
    const uint32_t q4 = warp & 3;               // TMEM lane quarter accessible to this warp
    long long e_wait = 0, e_ld = 0, e_math = 0, e_t0 = clock64(), e_g0 = 0;
    const bool eprof = kProf && warp == 5;
    if (eprof) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(e_g0));
    const uint32_t cq = warp >> 2;        // column group (kColsW wide) of the 256-wide tile
    int it = 0;
    for (int item = it_lo; item < it_hi; ++item, ++it) {
      int s, rb, jt, half;
      decode_item<kLF>(p, pi, item, s, rb, jt, half);
      const SimSeg& sg = p.seg[s];
      // a half tile holds its 128 columns in TMEM columns 0..127. FUSED / Q / RAW spread them
      // over all column groups (half the chunks per warp); STATS keeps its 64-column row
      // partials per warp, so there the groups past 128 columns idle
      const int tile_off = half < 0 ? 0 : half * (kPairN / 2);   // first column inside the 256-wide tile
      constexpr bool kSpreadHalf = kMode != kSimStats && kMode != kSimFused;
      const int cols_w = (half >= 0 && kSpreadHalf) ? kColsW / 2 : kColsW;   // this warp's columns
      const int chunks_w = cols_w / 32;
      const bool active = static_cast<int>(cq) * cols_w < (half < 0 ? kPairN : kPairN / 2);
      const uint32_t acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int warp_row0 = rb * kPairM + static_cast<int>(rank) * kCtaM + static_cast<int>(q4) * 32;
      const int r_loc = warp_row0 + static_cast<int>(lane);
      const bool row_ok = r_loc < sg.rows;
      const bool warp_rows_ok = warp_row0 + 32 <= sg.rows;
      const int g0 = sg.a_row0 + warp_row0;     // global index of lane 0's anchor
      const int gi = g0 + static_cast<int>(lane);
      const int colq = jt * kPairN + tile_off + static_cast<int>(cq) * cols_w;

      float2 rstat = make_float2(0.f, 0.f);
      float rk = 0.f, rbeta = 0.f, rc = 0.f, rf = 0.f;
      if (row_ok) {
        if constexpr (kStatsLike) rstat = sg.row_stat[r_loc];
        if constexpr (kMode == kSimQ) {
          rk = sg.row_kappa[r_loc];
          rbeta = sg.row_beta[r_loc];
          rc = sg.row_coef[r_loc];
          rf = sg.row_fac[r_loc];
        }
      }

      // every global load of the tile is issued before the accumulator wait (latency hidden)
      float bnd0 = 0.f, bnd1 = 0.f, bnd2 = 0.f;
      for (int k = 0; k < p.n_bounds; ++k) {
        bnd0 = fmaxf(bnd0, p.bounds[4 * k]);
        bnd1 = fmaxf(bnd1, p.bounds[4 * k + 1]);
        bnd2 = fmaxf(bnd2, p.bounds[4 * k + 2]);
      }
      float2 cst_all[kMode == kSimFused ? kChunksW : 1];
      if constexpr (kMode == kSimFused) {
#pragma unroll
        for (int h = 0; h < kChunksW; ++h) {
          const int jc = colq + 32 * h + static_cast<int>(lane);
          cst_all[h] = (h < chunks_w && jc < sg.cols) ? sg.col_stat[jc] : f2(0.f, 0.f);
        }
      }
      long long ta = eprof ? clock64() : 0;
      mbar_wait(&L.tfull[acc], acc_phase);
      long long tb = eprof ? clock64() : 0;
      if (eprof) e_wait += tb - ta;
      tc_fence_after();
      // safe_exp can only clamp if some exponent may exceed 60: |s| <= |E1|max |E2|max bounds it
      const float smax = sqrtf(bnd0 * bnd1) * 1.0001f;
      const uint32_t taddr = tmem_base + ((q4 * 32u) << 16) + acc * kPairN + cq * static_cast<uint32_t>(cols_w);
      float2 se2 = f2(0.f, 0.f), sye2 = f2(0.f, 0.f);
      float se = 0.f, sye = 0.f;
      uint32_t ncl = 0;
      int ps = 0;
      const float* par = nullptr;
      bool q_col_safe = false, q_fact = false;
      if constexpr (kMode == kSimQ) {
        ps = it % kSimPSlots;
        mbar_wait(&L.pfull[ps], (it / kSimPSlots) & 1);
        par = L.par + ps * (kSimPSlotBytes / 4) + tile_off + cq * cols_w;
        q_col_safe = 2.f * smax * bnd2 <= kClampLog2;
        // factorized form: 2^(s kappa) stays within [2^-63, 2^63] and fac within fp32 range
        q_fact = p.q_factor && __all_sync(0xffffffffu, rk * smax <= kFactMaxLog2);
      }
      const float row_kap = kMode == kSimQ ? rk : rstat.x;
      const float row_beta = kMode == kSimQ ? rbeta : rstat.y;
      const bool row_safe = !__any_sync(0xffffffffu, row_ok && fmaf(smax, row_kap, row_beta) > kClampLog2);
      // FUSED one-exponential form: 2^(s kappa) and 2^beta stay inside [2^-63, 2^63]
      const bool fused_ok = kMode == kSimFused && __all_sync(0xffffffffu, row_kap * smax <= kFactMaxLog2);
      // FUSED: [chunk][q4][32] column sums of this column group for the tile (parity buffer)
      float2* red = reinterpret_cast<float2*>(L.par) + ((it & 1) * (kEpi / 4) + static_cast<int>(cq)) * (kChunksW * 4 * 32);
      if (!active) {   // half tile, columns beyond it: hand the buffer back at once
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (rank == 0) mbar_arrive(&L.tempty[acc]);
          else mbar_arrive_cluster(&L.tempty[acc], 0);
        }
      }
#pragma unroll 1
      for (int h = 0; h < (active ? chunks_w : 0); ++h) {
        uint32_t rr[kMode == kSimFused ? 1 : 32];
        if constexpr (kMode != kSimFused) {
          tmem_ld_32x32b_x32(taddr + 32 * h, rr);
          tmem_ld_wait();
        }
        if (kMode != kSimFused && h == chunks_w - 1) {   // the tile is in registers: hand the TMEM buffer back
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (rank == 0) mbar_arrive(&L.tempty[acc]);
            else mbar_arrive_cluster(&L.tempty[acc], 0);
          }
        }
        const int col0 = colq + 32 * h;
        const bool interior = (col0 + 32 <= sg.cols) && !(col0 < g0 + 32 && g0 < col0 + 32);
        if constexpr (kMode == kSimRaw) {
          if (row_ok) {
            float* dst = raw_out + static_cast<size_t>(r_loc) * sg.cols;
#pragma unroll
            for (int k = 0; k < 32; ++k)
              if (col0 + k < sg.cols) dst[col0 + k] = __uint_as_float(rr[k]);
          }
        } else if constexpr (kMode == kSimStats) {
          bool fast = interior && warp_rows_ok;
          if (p.exact_bounds) {   // the chunk's row maxima decide whether safe_exp can clamp
            if (fast) {
              float mx = __uint_as_float(rr[0]);
#pragma unroll
              for (int k = 1; k < 32; ++k) mx = fmaxf(mx, __uint_as_float(rr[k]));
              fast = __all_sync(0xffffffffu, fmaf(mx, rstat.x, rstat.y) <= kClampLog2);
            }
          } else {
            fast = fast && row_safe;
          }
          if (fast) stats_fast(rr, rstat.x, rstat.y, se2, sye2);
          else stats_masked(rr, rstat.x, rstat.y, col0, sg.cols, gi, row_ok, se, sye, ncl);
        } else if constexpr (kMode == kSimFused) {
          // column anchor of this lane (the statistics it collects) and its parameters
          const int jc = col0 + static_cast<int>(lane);
          float2 cst = cst_all[0];
#pragma unroll
          for (int q = 1; q < kChunksW; ++q)
            if (h == q) cst = cst_all[q];
          const bool col_safe = !__any_sync(0xffffffffu, jc < sg.cols && fmaf(smax, cst.x, cst.y) > kClampLog2);
          const bool fast = p.fuse_fast && interior && warp_rows_ok && row_safe && col_safe && fused_ok;
          auto release_tmem = [&]() {   // the tile is in registers: release the TMEM buffer
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              if (rank == 0) mbar_arrive(&L.tempty[acc]);
              else mbar_arrive_cluster(&L.tempty[acc], 0);
            }
          };
          float ce = 0.f, cye = 0.f;
          if (fast) {
            // two 16-column halves (x / z x of 16 columns stay within the 16-warp register
            // budget); lanes 0-15 keep the first half's column sums, lanes 16-31 the second's
            float c0x, c0zx, c1x, c1zx;
            uint32_t r16[16];
            tmem_ld_32x32b_x16(taddr + 32 * h, r16);
            tmem_ld_wait();
            fused_fast16(r16, rstat.x, se2, sye2, lane, c0x, c0zx);
            tmem_ld_32x32b_x16(taddr + 32 * h + 16, r16);
            tmem_ld_wait();
            if (h == chunks_w - 1) release_tmem();
            fused_fast16(r16, rstat.x, se2, sye2, lane, c1x, c1zx);
            ce = lane < 16 ? c0x : c1x;
            cye = lane < 16 ? c0zx : c1zx;
          } else {
            // per 16-column half: exact bounds from the tile values themselves (the norm bound
            // smax is loose at small tau / for per-anchor temperatures): the row maxima and the
            // half's maximum / maximum |s| decide whether any exponent can reach the clamp and
            // whether the one-exponential form's range (kappa |s| <= 63, |beta| <= 63) holds
#pragma unroll 1
            for (int hh = 0; hh < 2; ++hh) {
              uint32_t r16[16];
              tmem_ld_32x32b_x16(taddr + 32 * h + 16 * hh, r16);
              tmem_ld_wait();
              if (hh == 1 && h == chunks_w - 1) release_tmem();
              int mode = 0;   // 0: masked exact path, 1: one exponential, 2: two exponentials
              if (interior && warp_rows_ok) {
                float mx = __uint_as_float(r16[0]), am = fabsf(mx);
#pragma unroll
                for (int k = 1; k < 16; ++k) {
                  const float v = __uint_as_float(r16[k]);
                  mx = fmaxf(mx, v);
                  am = fmaxf(am, fabsf(v));
                }
                float M = mx, A = am;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                  M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
                  A = fmaxf(A, __shfl_xor_sync(0xffffffffu, A, o));
                }
                const bool col_in = (lane >> 4) == static_cast<uint32_t>(hh);   // lanes of this half's columns
                if (__all_sync(0xffffffffu, fmaf(mx, rstat.x, rstat.y) <= kClampLog2 &&
                                                (!col_in || fmaf(M, cst.x, cst.y) <= kClampLog2))) {
                  const bool one = p.fuse_fast && __all_sync(0xffffffffu, rstat.x * A <= kFactMaxLog2 &&
                                                                            fabsf(rstat.y) <= kFactMaxLog2 &&
                                                                            (!col_in || fabsf(cst.y) <= kFactMaxLog2));
                  mode = one ? 1 : 2;
                }
              }
              if (mode == 0) {
#pragma unroll
                for (int q = 0; q < 2; ++q) {
                  uint32_t r8[8];
#pragma unroll
                  for (int k = 0; k < 8; ++k) r8[k] = r16[8 * q + k];
                  fused_masked(r8, rstat, sg.col_stat, col0 + 16 * hh + 8 * q, sg.cols, gi, row_ok, lane, 2 * hh + q,
                               se, sye, ncl, ce, cye);
                }
                continue;
              }
              float cx, cy;
              if (mode == 1) {   // raw {sum x, sum z x} -> {sum e, sum y e} with 2^beta_j of the lane's column
                fused_fast16(r16, rstat.x, se2, sye2, lane, cx, cy);
                const float sc = ex2_approx(cst.y);
                cy = sc * fmaf(cst.y, cx, cy);
                cx = sc * cx;
              } else {
                float2 re = f2(0.f, 0.f), rye = f2(0.f, 0.f);
                if (p.fuse_fast) fused_2e16<true>(r16, rstat, cst, 16 * hh, lane, re, rye, cx, cy);
                else fused_2e16<false>(r16, rstat, cst, 16 * hh, lane, re, rye, cx, cy);
                se += re.x + re.y;   // already {sum e, sum y e}
                sye += rye.x + rye.y;
              }
              if ((lane >> 4) == static_cast<uint32_t>(hh)) {
                ce = cx;
                cye = cy;
              }
            }
          }
          if (fast) {   // raw {sum x, sum z x} -> {sum e, sum y e} with 2^beta_j (|beta_j| <= 63)
            const float sc = ex2_approx(cst.y);
            cye = sc * fmaf(cst.y, ce, cye);
            ce = sc * ce;
          }
          // this warp's 32-row column sums -> shared memory; the tile's four lane-quarter warps
          // of this column group combine them after the chunk loop
          red[(h * 4 + static_cast<int>(q4)) * 32 + lane] = f2(ce, cye);
          if (h & 1) {   // 64 columns done: one row partial per (row, column quarter)
            // fast-path row raw sums {sum x, sum z x} -> e = 2^beta_i x, y e = (z + beta_i) e
            const float sc = ex2_approx(rstat.y);
            const float rx = se2.x + se2.y, rzx = sye2.x + sye2.y;
            const float sxe = sc * fmaf(rstat.y, rx, rzx) + sye;
            const int quarter = (tile_off + static_cast<int>(cq) * cols_w + 32 * h) / 64;
            if (row_ok)
              sg.partial[static_cast<size_t>(r_loc) * (p.n_jt * 4) + jt * 4 + quarter] = make_float2(se + sc * rx, sxe);
            se2 = f2(0.f, 0.f); sye2 = f2(0.f, 0.f); se = 0.f; sye = 0.f;
          }
        } else {  // kSimQ
          uint32_t packed[16];
          const float* kc = par + 32 * h;
          bool safe = interior && row_safe && q_col_safe;
          bool fact = safe && q_fact;
          if (interior && !fact) {
            // exact bounds from this chunk's values (the norm bounds are loose at small tau): no
            // exponent reaches the clamp, and the one-exponential range holds (kappa |s| <= 63,
            // |beta| <= 63 for the row and the 32 column anchors; column lane's parameters)
            float mx = __uint_as_float(rr[0]), am = fabsf(mx);
#pragma unroll
            for (int k = 1; k < 32; ++k) {
              const float v = __uint_as_float(rr[k]);
              mx = fmaxf(mx, v);
              am = fmaxf(am, fabsf(v));
            }
            float M = mx, A = am;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
              A = fmaxf(A, __shfl_xor_sync(0xffffffffu, A, o));
            }
            const float kj = kc[lane], bj = kc[kPairN + lane];
            safe = __all_sync(0xffffffffu, fmaf(mx, rk, rbeta) <= kClampLog2 && fmaf(M, kj, bj) <= kClampLog2);
            fact = safe && p.q_factor &&
                   __all_sync(0xffffffffu, rk * A <= kFactMaxLog2 && fabsf(rbeta) <= kFactMaxLog2 && fabsf(bj) <= kFactMaxLog2);
          }
          if (fact)
            q_chunk_fact(rr, rk, rf, kc + 3 * kPairN, packed);
          else if (safe)
            q_chunk<false>(rr, rk, rbeta, rc, kc, kc + kPairN, kc + 2 * kPairN, col0, sg.cols, gi, packed);
          else
            q_chunk<true>(rr, rk, rbeta, rc, kc, kc + kPairN, kc + 2 * kPairN, col0, sg.cols, gi, packed);
          if (col0 < p.ldq) {
            // 32 rows x 64 B through 64-byte-swizzled staging -> one TMA tile store (rows past
            // the segment and columns past ldq are clipped by the tensor map)
            uint8_t* stg = L.qout + warp * kSimStageOutQ;
            if (lane == 0) bulk_wait_read0();
            __syncwarp();
            uint8_t* rowp = stg + lane * 64;
            const uint32_t sw = (lane >> 1) & 3;
#pragma unroll
            for (int v4 = 0; v4 < 4; ++v4)
              *reinterpret_cast<uint4*>(rowp + ((v4 ^ sw) << 4)) =
                  make_uint4(packed[4 * v4], packed[4 * v4 + 1], packed[4 * v4 + 2], packed[4 * v4 + 3]);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_store_2d(s ? &mapQo1 : &mapQo0, stg, col0, warp_row0);
              bulk_commit();
            }
          }
        }
      }
      if constexpr (kMode == kSimFused) {
        // column partials: the four lane-quarter warps of the column group add their 32-row sums
        // in fixed order (q4 = 0..3), warp q4 taking chunk q4 -> one partial per (CTA, column),
        // a quarter of the partials the per-anchor kernel reads. One named barrier per tile;
        // the buffer alternates with the tile parity (the next tile's barrier orders the reuse).
        if (active) {
          named_bar_sync(1 + cq, 128);
          if (static_cast<int>(q4) < chunks_w) {
            float2 v = red[(q4 * 4 + 0) * 32 + lane];
#pragma unroll
            for (int q = 1; q < 4; ++q) {
              const float2 w = red[(q4 * 4 + q) * 32 + lane];
              v.x += w.x;
              v.y += w.y;
            }
            const int col0 = colq + 32 * static_cast<int>(q4);
            if (col0 + static_cast<int>(lane) < sg.cols)
              p.col_partial[(static_cast<size_t>(col0 >> 5) * p.n_slots + (rb * 2 + rank)) * 32 + lane] = v;
          }
        }
      }
      long long tc = eprof ? clock64() : 0;
      if constexpr (kMode == kSimFused) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ncl += __shfl_xor_sync(0xffffffffu, ncl, o);
        if (lane == 0 && ncl) atomicAdd(p.clamps, static_cast<unsigned long long>(ncl));
      }
      if constexpr (kMode == kSimStats) {
        const float sxe = sye2.x + sye2.y + sye;   // sum y e; the table kernel divides by kappa
        se += se2.x + se2.y;
        if (row_ok && active)
          sg.partial[static_cast<size_t>(r_loc) * (p.n_jt * 4) + jt * 4 + tile_off / 64 + cq] = make_float2(se, sxe);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ncl += __shfl_xor_sync(0xffffffffu, ncl, o);
        if (lane == 0 && ncl) atomicAdd(p.clamps, static_cast<unsigned long long>(ncl));
      }
      if constexpr (kMode == kSimQ) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&L.pempty[ps]);
      }
      if (eprof) e_math += clock64() - tc;
    }
    if (eprof && lane == 0 && rank == 0) {   // epilogue counters of one warp per pair
      long long* o = p.dbg_out + 1024 + pair * 8;
      o[0] = clock64() - e_t0; o[1] = e_wait; o[2] = e_ld; o[3] = e_math;
      o[4] = e_g0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(o[5]));   // epilogue loop end (ns)
    }
  }

  if constexpr (kMode == kSimQ) {
    if (warp < kProdWarp && lane == 0) bulk_wait0();
  }
  __syncwarp();   // single-thread producer / MMA roles reconverge before the aligned cluster barrier
  long long g_work_end = 0;
  if (kProf) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_work_end));
  tc_fence_before();
  cluster_sync();
  if (warp == 0) tmem_dealloc<2>(tmem_base, 512);
  if (kProf && threadIdx.x == 0) {
    long long g_exit;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_exit));
    long long* o = p.dbg_out + 2048 + blockIdx.x * 4;   // per-CTA timeline (ns)
    o[0] = g_entry; o[1] = g_work_end; o[2] = g_exit;
  }
}

cudaError_t sim_set_smem() {
  cudaError_t e = cudaFuncSetAttribute(sim_tile_kernel<kSimStats>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSimSmemBytes);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(sim_tile_kernel<kSimQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSimSmemBytes);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(sim_tile_kernel<kSimRaw>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSimSmemBytes);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(sim_tile_kernel<kSimFused>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSimSmemBytes);
  return e;
}

cudaError_t sim_attributes(int mode, cudaFuncAttributes* a) {
  return mode == kSimQ ? cudaFuncGetAttributes(a, sim_tile_kernel<kSimQ>) : cudaFuncGetAttributes(a, sim_tile_kernel<kSimStats>);
}

cudaError_t launch_sim(int mode, const SimParams& p, const CUtensorMap* mapA, const CUtensorMap* mapB,
                       const CUtensorMap* mapQout, int grid, cudaStream_t s, float* raw_out, bool pdl) {
  const CUtensorMap& a1 = p.nseg > 1 ? mapA[1] : mapA[0];
  const CUtensorMap& b1 = p.nseg > 1 ? mapB[1] : mapB[0];
  const CUtensorMap& q0 = mapQout ? mapQout[0] : mapA[0];
  const CUtensorMap& q1 = mapQout ? (p.nseg > 1 ? mapQout[1] : mapQout[0]) : mapA[0];
  if (grid < 2) grid = 2;
  grid &= ~1;
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.dynamicSmemBytes = kSimSmemBytes;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  switch (mode) {
    case kSimStats:
      cfg.blockDim = dim3(SimCfg<kSimStats>::kThreads, 1, 1);
      return cudaLaunchKernelEx(&cfg, sim_tile_kernel<kSimStats>, p, mapA[0], mapB[0], a1, b1, q0, q1, raw_out);
    case kSimFused:
      cfg.blockDim = dim3(SimCfg<kSimFused>::kThreads, 1, 1);
      return cudaLaunchKernelEx(&cfg, sim_tile_kernel<kSimFused>, p, mapA[0], mapB[0], a1, b1, q0, q1, raw_out);
    case kSimQ:
      cfg.blockDim = dim3(SimCfg<kSimQ>::kThreads, 1, 1);
      return cudaLaunchKernelEx(&cfg, sim_tile_kernel<kSimQ>, p, mapA[0], mapB[0], a1, b1, q0, q1, raw_out);
    default:
      cfg.blockDim = dim3(SimCfg<kSimRaw>::kThreads, 1, 1);
      return cudaLaunchKernelEx(&cfg, sim_tile_kernel<kSimRaw>, p, mapA[0], mapB[0], a1, b1, q0, q1, raw_out);
  }
}

}  // namespace fc
