// gemm_kernel.cu -- weighted-gradient GEMM (FastCLIP pass 2b) for sm_100a.
//
//   dE1[L] = c (Q'_R  E2[G] - r o E2[L]),   dE2[L] = c (Q'_C  E1[G] - r o E1[L])
// (engine.cpp:77-121 regrouped: Q[i,j] = P1[i,j] + P2[j,i], r_i = a_i S1_i + b_i S2_i,
//  c = 1/(Bl (B-1))). A = Q' (bf16, K-major, written by the Q pass), B = E (bf16, N = d
// contiguous => MN-major UMMA operand), fp32 accumulation in TMEM. Persistent CTA pairs
// (cta_group::2, 256 x 256 pair tiles) over (segment, row block, column block, K split);
// split-K partials are reduced with vector fp32 atomics into a zeroed output.
#include "kernels.cuh"
#include "sm100.cuh"

namespace fc {

namespace {

struct GSmem {
  uint8_t* a;
  uint8_t* b;
  uint64_t* full;
  uint64_t* empty;
  uint64_t* tfull;
  uint64_t* tempty;
  uint32_t* tmem_ptr;
};

__device__ __forceinline__ GSmem gcarve(uint8_t* base) {
  GSmem L;
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

__device__ __forceinline__ void gdecode(const GemmParams& p, int item, int& s, int& mb, int& nb, int& ks) {
  const int per_seg0 = p.n_mb[0] * p.n_nb * p.n_split;
  s = item < per_seg0 ? 0 : 1;
  int local = item - (s ? per_seg0 : 0);
  // column block fastest: pairs running side by side read the same Q' rows and K range,
  // so the second read of each Q' tile is an L2 hit (Q' is streamed from HBM once).
  nb = local % p.n_nb;
  local /= p.n_nb;
  ks = local % p.n_split;
  mb = local / p.n_split;
}

}  // namespace

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    grad_gemm_kernel(const __grid_constant__ GemmParams p, const __grid_constant__ CUtensorMap mapQ0,
                     const __grid_constant__ CUtensorMap mapX0, const __grid_constant__ CUtensorMap mapQ1,
                     const __grid_constant__ CUtensorMap mapX1) {
  extern __shared__ uint8_t smem_raw[];
  const GSmem L = gcarve(smem_raw);
  const uint32_t warp = threadIdx.x / 32;
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x / 2;
  const int n_pairs = gridDim.x / 2;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&mapQ0);
    tma_prefetch(&mapX0);
    if (p.nseg > 1) {
      tma_prefetch(&mapQ1);
      tma_prefetch(&mapX1);
    }
  }
  if (warp == 1 && lane == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&L.full[i], 2);
      mbar_init(&L.empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&L.tfull[i], 1);
      mbar_init(&L.tempty[i], 2 * kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<2>(L.tmem_ptr, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *L.tmem_ptr;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (elect_one()) {
      uint32_t stage = 0, phase = 0;
      for (int item = pair; item < p.n_items; item += n_pairs) {
        int s, mb, nb, ks;
        gdecode(p, item, s, mb, nb, ks);
        const CUtensorMap* mq = s ? &mapQ1 : &mapQ0;
        const CUtensorMap* mx = s ? &mapX1 : &mapX0;
        const int a_row = mb * kPairM + static_cast<int>(rank) * kCtaM;
        const int n0 = nb * kPairN + static_cast<int>(rank) * (kPairN / 2);
        const int kb0 = ks * p.kb_per_split;
        const int kb1 = min(p.kb_total, kb0 + p.kb_per_split);
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&L.empty[stage], phase ^ 1);
          if (rank == 0)
            mbar_arrive_expect_tx(&L.full[stage], 2 * (kStageBytesA + kStageBytesB));
          else
            mbar_arrive_cluster(&L.full[stage], 0);
          uint8_t* sb = L.b + stage * kStageBytesB;
          if (p.seg[s].a_mn_major) {
            // A = Q^T: two 64(M) x 64(K) swizzle atoms of the row-major Q (K = rows of Q)
            uint8_t* sa = L.a + stage * kStageBytesA;
            tma_load_2d_pair(mq, &L.full[stage], sa, a_row, kb * kBlockK);
            tma_load_2d_pair(mq, &L.full[stage], sa + kStageBytesA / 2, a_row + 64, kb * kBlockK);
          } else {
            tma_load_2d_pair(mq, &L.full[stage], L.a + stage * kStageBytesA, kb * kBlockK, a_row);
          }
          // MN-major B: two 64(N) x 64(K) swizzle atoms for this CTA's 128 columns of N.
          tma_load_2d_pair(mx, &L.full[stage], sb, n0, kb * kBlockK);
          tma_load_2d_pair(mx, &L.full[stage], sb + kStageBytesB / 2, n0 + 64, kb * kBlockK);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader) =====================
    if (rank == 0) {
      constexpr uint32_t idesc_k = make_idesc_bf16(kPairM, kPairN, 0, 1);
      constexpr uint32_t idesc_mn = make_idesc_bf16(kPairM, kPairN, 1, 1);
      uint32_t stage = 0, phase = 0;
      int it = 0;
      for (int item = pair; item < p.n_items; item += n_pairs, ++it) {
        int s, mb, nb, ks;
        gdecode(p, item, s, mb, nb, ks);
        const int kb0 = ks * p.kb_per_split;
        const int kb1 = min(p.kb_total, kb0 + p.kb_per_split);
        const bool a_mn = p.seg[s].a_mn_major != 0;
        const uint32_t idesc = a_mn ? idesc_mn : idesc_k;
        const uint32_t acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&L.tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kPairN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&L.full[stage], phase);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t a0 = smem_u32(L.a + stage * kStageBytesA);
            const uint32_t b0 = smem_u32(L.b + stage * kStageBytesB);
#pragma unroll
            for (int k = 0; k < kBlockK / 16; ++k) {
              const uint64_t ad = a_mn ? make_sdesc_sw128(a0 + k * 2048, kStageBytesA / 2, 1024)
                                       : make_sdesc_sw128(a0 + k * 32, 0, 1024);
              // MN-major SW128: 16 K rows of 128 B per UMMA_K; LBO = next 64-wide N atom.
              const uint64_t bd = make_sdesc_sw128(b0 + k * 2048, kStageBytesB / 2, 1024);
              mma_bf16_pair(d_tmem, ad, bd, idesc, (kb != kb0) || (k != 0));
            }
            mma_commit_pair(&L.empty[stage], 0x3);
            if (kb == kb1 - 1) mma_commit_pair(&L.tfull[acc], 0x3);
          }
          __syncwarp();
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else {
    // ===================== epilogue =====================
    const uint32_t q4 = warp & 3;
    const uint32_t half = (warp - 2) >> 2;
    const int row_in_cta = static_cast<int>(q4 * 32 + lane);
    int it = 0;
    for (int item = pair; item < p.n_items; item += n_pairs, ++it) {
      int s, mb, nb, ks;
      gdecode(p, item, s, mb, nb, ks);
      const GemmSeg& sg = p.seg[s];
      const uint32_t acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int r_loc = mb * kPairM + static_cast<int>(rank) * kCtaM + row_in_cta;
      const bool row_ok = r_loc < sg.rows;
      const float rr = (row_ok && ks == 0) ? sg.r[r_loc] : 0.f;
      const __nv_bfloat16* xrow = sg.x + static_cast<size_t>(sg.x_row0 + (row_ok ? r_loc : 0)) * p.d;
      float* orow = sg.out + static_cast<size_t>(row_ok ? r_loc : 0) * p.d;
      mbar_wait(&L.tfull[acc], acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        const int col0 = nb * kPairN + static_cast<int>(half) * 128 + c * 32;
        const uint32_t taddr = tmem_base + ((q4 * 32u) << 16) + acc * kPairN + half * 128u + c * 32u;
        uint32_t r[32];
        tmem_ld_32x32b_x32(taddr, r);
        tmem_ld_wait();
        if (row_ok && col0 < p.d) {
          float v[32];
#pragma unroll
          for (int k = 0; k < 32; ++k) v[k] = __uint_as_float(r[k]);
          if (ks == 0) {
            const uint4* xs = reinterpret_cast<const uint4*>(xrow + col0);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              if (col0 + 8 * q >= p.d) break;  // d % 8 == 0: groups of 8 are all-in or all-out
              const uint4 w = __ldg(xs + q);
              const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
              for (int t = 0; t < 4; ++t) {
                const __nv_bfloat162 h2 = *reinterpret_cast<const __nv_bfloat162*>(&ww[t]);
                const float2 f = __bfloat1622float2(h2);
                v[q * 8 + 2 * t] -= rr * f.x;
                v[q * 8 + 2 * t + 1] -= rr * f.y;
              }
            }
          }
          float4* dst = reinterpret_cast<float4*>(orow + col0);
          if (p.n_split == 1) {
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (col0 + 4 * q < p.d)
                dst[q] = make_float4(p.scale * v[4 * q], p.scale * v[4 * q + 1], p.scale * v[4 * q + 2], p.scale * v[4 * q + 3]);
          } else {
#pragma unroll
            for (int q = 0; q < 8; ++q)
              if (col0 + 4 * q < p.d)
                atomicAdd(dst + q, make_float4(p.scale * v[4 * q], p.scale * v[4 * q + 1], p.scale * v[4 * q + 2],
                                             p.scale * v[4 * q + 3]));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (rank == 0) mbar_arrive(&L.tempty[acc]);
        else mbar_arrive_cluster(&L.tempty[acc], 0);
      }
    }
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 2) tmem_dealloc<2>(tmem_base, 512);
}

cudaError_t gemm_set_smem() {
  return cudaFuncSetAttribute(grad_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
}

cudaError_t launch_gemm(const GemmParams& p, const CUtensorMap* mapQ, const CUtensorMap* mapX, int grid,
                        cudaStream_t s) {
  const CUtensorMap& q1 = p.nseg > 1 ? mapQ[1] : mapQ[0];
  const CUtensorMap& x1 = p.nseg > 1 ? mapX[1] : mapX[0];
  if (grid < 2) grid = 2;
  grid &= ~1;
  grad_gemm_kernel<<<grid, kThreads, kSmemBytes, s>>>(p, mapQ[0], mapX[0], q1, x1);
  return cudaGetLastError();
}

}  // namespace fc
