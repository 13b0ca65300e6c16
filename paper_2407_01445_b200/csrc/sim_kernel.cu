// sim_kernel.cu -- fused similarity-tile kernel (FastCLIP pass 1 and pass 2a) for sm_100a.
//
// A persistent CTA pair (cluster of 2, tcgen05 cta_group::2) walks (segment, row block,
// column tile) items. Per item the pair computes one 256 x 256 tile of S' = A B^T (K = d)
// into TMEM with bf16 UMMA (M = 256 split 128/128 over the pair, N = 256 with each CTA
// supplying half of B), double-buffered so the epilogue of tile t overlaps the MMAs of t+1.
// The epilogue never writes S:
//   STATS: per anchor row i, over the tile's columns j != i,
//            e = exp(min((s_ij - s_ii)/t_i, 60))    (safe_exp, losses.cpp:22-28)
//            sum e, sum (s_ij - s_ii) e             (engine.cpp:151-176, :182-204)
//          -> one float2 partial per (row, column half-tile), reduced in fixed order later.
//   Q:     Q'_ij = coef_i e_row(i,j) + coef_j e_col(i,j) (Q[i,j] = P1[i,j] + P2[j,i] of
//          engine.cpp:91-118) -> bf16 tile of the weight matrix for the gradient GEMM.
// Warp roles: w0 TMA producer, w1 MMA issuer (leader CTA), w2..w9 epilogue (2 warps per
// TMEM lane quarter, one per column half).
#include "kernels.cuh"
#include "sm100.cuh"

namespace fc {

namespace {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kClampLog2 = 60.0f * 1.4426950408889634f;  // kExpClampMax in the log2 domain

struct SmemLayout {
  uint8_t* a;   // kStages x 16 KB
  uint8_t* b;   // kStages x 16 KB
  uint64_t* full;
  uint64_t* empty;
  uint64_t* tfull;
  uint64_t* tempty;
  uint32_t* tmem_ptr;
};

__device__ __forceinline__ SmemLayout carve(uint8_t* base) {
  SmemLayout L;
  uint8_t* p = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(base) + 1023) & ~uintptr_t(1023));
  L.a = p;
  L.b = p + kStages * kStageBytesA;
  uint64_t* bars = reinterpret_cast<uint64_t*>(L.b + kStages * kStageBytesB);
  L.full = bars;
  L.empty = bars + kStages;
  L.tfull = bars + 2 * kStages;
  L.tempty = bars + 2 * kStages + 2;
  L.tmem_ptr = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 4);
  return L;
}

__device__ __forceinline__ void decode_item(const SimParams& p, int item, int& s, int& rb, int& jt) {
  const int n0 = p.n_rb[0] * p.n_jt;
  s = item < n0 ? 0 : 1;
  const int local = item - (s ? n0 : 0);
  rb = local / p.n_jt;
  jt = local % p.n_jt;
}

}  // namespace

template <int kMode>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    sim_tile_kernel(const __grid_constant__ SimParams p, const __grid_constant__ CUtensorMap mapA0,
                    const __grid_constant__ CUtensorMap mapB0, const __grid_constant__ CUtensorMap mapA1,
                    const __grid_constant__ CUtensorMap mapB1, float* __restrict__ raw_out) {
  extern __shared__ uint8_t smem_raw[];
  const SmemLayout L = carve(smem_raw);
  const uint32_t warp = threadIdx.x / 32;
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x / 2;
  const int n_pairs = gridDim.x / 2;
  const int nkb = (p.d + kBlockK - 1) / kBlockK;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&mapA0);
    tma_prefetch(&mapB0);
    if (p.nseg > 1) {
      tma_prefetch(&mapA1);
      tma_prefetch(&mapB1);
    }
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&L.full[i], 2);   // leader's expect_tx arrive + peer's remote arrive
      mbar_init(&L.empty[i], 1);  // MMA commit (multicast to both CTAs)
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&L.tfull[i], 1);                 // MMA commit (multicast)
      mbar_init(&L.tempty[i], 2 * kEpiWarps);    // one arrive per epilogue warp of the pair
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<2>(L.tmem_ptr, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *L.tmem_ptr;

  if (warp == 0) {
    // ===================== TMA producer (both CTAs) =====================
    if (elect_one()) {
      uint32_t stage = 0, phase = 0;
      for (int item = pair; item < p.n_items; item += n_pairs) {
        int s, rb, jt;
        decode_item(p, item, s, rb, jt);
        const CUtensorMap* ma = s ? &mapA1 : &mapA0;
        const CUtensorMap* mb = s ? &mapB1 : &mapB0;
        const int a_row = p.seg[s].a_row0 + rb * kPairM + static_cast<int>(rank) * kCtaM;
        const int b_row = jt * kPairN + static_cast<int>(rank) * (kPairN / 2);
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&L.empty[stage], phase ^ 1);
          if (rank == 0)
            mbar_arrive_expect_tx(&L.full[stage], 2 * (kStageBytesA + kStageBytesB));
          else
            mbar_arrive_cluster(&L.full[stage], 0);
          tma_load_2d_pair(ma, &L.full[stage], L.a + stage * kStageBytesA, kb * kBlockK, a_row);
          tma_load_2d_pair(mb, &L.full[stage], L.b + stage * kStageBytesB, kb * kBlockK, b_row);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA only) =====================
    if (rank == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(kPairM, kPairN, 0, 0);
      uint32_t stage = 0, phase = 0;
      int it = 0;
      for (int item = pair; item < p.n_items; item += n_pairs, ++it) {
        const uint32_t acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&L.tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kPairN;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&L.full[stage], phase);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t a0 = smem_u32(L.a + stage * kStageBytesA);
            const uint32_t b0 = smem_u32(L.b + stage * kStageBytesB);
#pragma unroll
            for (int k = 0; k < kBlockK / 16; ++k) {
              const uint64_t ad = make_sdesc_sw128(a0 + k * 32, 0, 1024);
              const uint64_t bd = make_sdesc_sw128(b0 + k * 32, 0, 1024);
              mma_bf16_pair(d_tmem, ad, bd, idesc, (kb | k) != 0);
            }
            mma_commit_pair(&L.empty[stage], 0x3);
            if (kb == nkb - 1) mma_commit_pair(&L.tfull[acc], 0x3);
          }
          __syncwarp();
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else {
    // ===================== epilogue (both CTAs) =====================
    const uint32_t q4 = warp & 3;               // TMEM lane quarter of this warp
    const uint32_t half = (warp - 2) >> 2;      // column half of the 256-wide tile
    const int row_in_cta = static_cast<int>(q4 * 32 + lane);
    int it = 0;
    for (int item = pair; item < p.n_items; item += n_pairs, ++it) {
      int s, rb, jt;
      decode_item(p, item, s, rb, jt);
      const SimSeg& sg = p.seg[s];
      const uint32_t acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int r_loc = rb * kPairM + static_cast<int>(rank) * kCtaM + row_in_cta;
      const bool row_ok = r_loc < sg.rows;
      const int gi = sg.a_row0 + r_loc;
      float2 rstat = make_float2(0.f, 0.f);
      float4 rpar = make_float4(0.f, 0.f, 0.f, 0.f);
      if (row_ok) {
        if constexpr (kMode == kSimStats) rstat = sg.row_stat[r_loc];
        if constexpr (kMode == kSimQ) rpar = sg.row_par[r_loc];
      }
      float sum_e = 0.f, sum_xe = 0.f;
      uint32_t nclamp = 0;

      mbar_wait(&L.tfull[acc], acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        const int col0 = jt * kPairN + static_cast<int>(half) * 128 + c * 32;
        const uint32_t taddr = tmem_base + ((q4 * 32u) << 16) + acc * kPairN + half * 128u + c * 32u;
        uint32_t r[32];
        tmem_ld_32x32b_x32(taddr, r);
        tmem_ld_wait();
        if constexpr (kMode == kSimRaw) {
          if (row_ok) {
            float* dst = raw_out + static_cast<size_t>(r_loc) * sg.cols;
#pragma unroll
            for (int k = 0; k < 32; ++k)
              if (col0 + k < sg.cols) dst[col0 + k] = __uint_as_float(r[k]);
          }
        } else if constexpr (kMode == kSimStats) {
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            const int j = col0 + k;
            const float x = __uint_as_float(r[k]) - rstat.x;
            float y = x * rstat.y;
            const bool clamped = y > kClampLog2;
            y = fminf(y, kClampLog2);
            const float e = ex2_approx(y);
            const bool ok = row_ok && (j < sg.cols) && (j != gi);
            sum_e += ok ? e : 0.f;
            sum_xe += ok ? x * e : 0.f;
            nclamp += (ok && clamped) ? 1u : 0u;
          }
        } else {  // kSimQ
          if (row_ok && col0 < p.ldq) {
            uint32_t packed[16];
#pragma unroll
            for (int k = 0; k < 32; k += 2) {
              float qv[2];
#pragma unroll
              for (int u = 0; u < 2; ++u) {
                const int j = col0 + k + u;
                const float sv = __uint_as_float(r[k + u]);
                const bool ok = (j < sg.cols) && (j != gi);
                const float4 cp = ok ? __ldg(&sg.col_par[j]) : make_float4(0.f, 0.f, 0.f, 0.f);
                const float yr = fminf((sv - rpar.x) * rpar.y, kClampLog2);
                const float yc = fminf((sv - cp.x) * cp.y, kClampLog2);
                const float v = rpar.z * ex2_approx(yr) + cp.z * ex2_approx(yc);
                qv[u] = ok ? v : 0.f;
              }
              __nv_bfloat162 h2 = __floats2bfloat162_rn(qv[0], qv[1]);
              packed[k / 2] = *reinterpret_cast<uint32_t*>(&h2);
            }
            uint4* dst = reinterpret_cast<uint4*>(sg.q + static_cast<size_t>(r_loc) * p.ldq + col0);
#pragma unroll
            for (int v4 = 0; v4 < 4; ++v4)
              dst[v4] = make_uint4(packed[4 * v4], packed[4 * v4 + 1], packed[4 * v4 + 2], packed[4 * v4 + 3]);
          }
        }
      }
      // TMEM buffer drained: hand it back to the MMA warp of the leader CTA.
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (rank == 0) mbar_arrive(&L.tempty[acc]);
        else mbar_arrive_cluster(&L.tempty[acc], 0);
      }
      if constexpr (kMode == kSimStats) {
        if (row_ok) sg.partial[static_cast<size_t>(r_loc) * (p.n_jt * 2) + jt * 2 + half] = make_float2(sum_e, sum_xe);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) nclamp += __shfl_xor_sync(0xffffffffu, nclamp, o);
        if (lane == 0 && nclamp) atomicAdd(p.clamps, static_cast<unsigned long long>(nclamp));
      }
    }
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 2) tmem_dealloc<2>(tmem_base, 512);
}

cudaError_t launch_sim(int mode, const SimParams& p, const CUtensorMap* mapA, const CUtensorMap* mapB, int grid,
                       cudaStream_t s, float* raw_out) {
  const CUtensorMap& a1 = p.nseg > 1 ? mapA[1] : mapA[0];
  const CUtensorMap& b1 = p.nseg > 1 ? mapB[1] : mapB[0];
  if (grid < 2) grid = 2;
  grid &= ~1;
  cudaError_t e;
  switch (mode) {
    case kSimStats:
      e = cudaFuncSetAttribute(sim_tile_kernel<kSimStats>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
      if (e != cudaSuccess) return e;
      sim_tile_kernel<kSimStats><<<grid, kThreads, kSmemBytes, s>>>(p, mapA[0], mapB[0], a1, b1, raw_out);
      break;
    case kSimQ:
      e = cudaFuncSetAttribute(sim_tile_kernel<kSimQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
      if (e != cudaSuccess) return e;
      sim_tile_kernel<kSimQ><<<grid, kThreads, kSmemBytes, s>>>(p, mapA[0], mapB[0], a1, b1, raw_out);
      break;
    default:
      e = cudaFuncSetAttribute(sim_tile_kernel<kSimRaw>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
      if (e != cudaSuccess) return e;
      sim_tile_kernel<kSimRaw><<<grid, kThreads, kSmemBytes, s>>>(p, mapA[0], mapB[0], a1, b1, raw_out);
      break;
  }
  return cudaGetLastError();
}

}  // namespace fc
