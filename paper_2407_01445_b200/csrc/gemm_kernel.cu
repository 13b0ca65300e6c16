// gemm_kernel.cu -- weighted-gradient GEMM (FastCLIP pass 2b) for sm_100a.
//
//   dE1[L] = c (Q'_R  E2[G] - r o E2[L]),   dE2[L] = c (Q'_C  E1[G] - r o E1[L])
// (engine.cpp:77-121 regrouped: Q[i,j] = P1[i,j] + P2[j,i], r_i = a_i S1_i + b_i S2_i,
//  c = 1/(Bl (B-1))). A = Q' (bf16, K-major, written by the Q pass; at K = 1 the dE2 GEMM
// reads Q^T through an MN-major A operand), B = E (bf16, N = d contiguous => MN-major UMMA
// operand), fp32 accumulation in TMEM, CTA pairs (cta_group::2, 256 x 256 pair tiles).
//
// Schedule (hybrid data-parallel + stream-K): the first floor(T/P)*P tiles are processed
// whole, one tile per pair per round, and stored directly; the k-blocks of the remaining
// T mod P tiles are split evenly over all P pairs (contiguous k ranges) and reduced with
// vector fp32 atomics into a pre-zeroed output. Every pair therefore runs the same number
// of k-blocks (+-1) whatever T is.
#include "kernels.cuh"
#include "sm100.cuh"

namespace fc {

namespace {

struct GSmem {
  uint8_t* a;
  uint8_t* b;
  uint8_t* out;   // kEpiWarps x 4 KB epilogue staging (TMA store / reduce-add source)
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
  L.out = L.b + kStages * kStageBytesB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(L.out + kEpiWarps * kGemmStageOut);
  L.full = bars;
  L.empty = bars + kStages;
  L.tfull = bars + 2 * kStages;
  L.tempty = bars + 2 * kStages + 2;
  L.tmem_ptr = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 4);
  return L;
}

// tile -> (segment, row block, column block); column block fastest so that pairs running
// side by side read the same Q' rows (the second read of each Q' tile hits L2).
__device__ __forceinline__ void tile_decode(const GemmParams& p, int t, int& s, int& mb, int& nb) {
  const int per_seg0 = p.n_mb[0] * p.n_nb;
  s = t < per_seg0 ? 0 : 1;
  const int local = t - (s ? per_seg0 : 0);
  nb = local % p.n_nb;
  mb = local / p.n_nb;
}

// The pair's sequence of (tile, k-block range, atomic?) work segments.
struct SegIter {
  int pair, n_pairs, T, KB, dp_tiles;   // dp_tiles = floor(T / P) * P
  int t;                                // next data-parallel tile
  long long u, u1;                      // stream-K unit range (units = remainder tile k-blocks)
  __device__ SegIter(const GemmParams& p, int pair_, int n_pairs_) {
    pair = pair_;
    n_pairs = n_pairs_;
    T = p.n_tiles;
    KB = p.kb_total;
    dp_tiles = (T / n_pairs) * n_pairs;
    t = pair;
    const long long U = static_cast<long long>(T - dp_tiles) * KB;
    u = U * pair / n_pairs;
    u1 = U * (pair + 1) / n_pairs;
  }
  __device__ bool next(int& tile, int& kb0, int& kb1, bool& atomic) {
    if (t < dp_tiles) {
      tile = t;
      kb0 = 0;
      kb1 = KB;
      atomic = false;
      t += n_pairs;
      return true;
    }
    if (u >= u1) return false;
    tile = dp_tiles + static_cast<int>(u / KB);
    kb0 = static_cast<int>(u % KB);
    kb1 = static_cast<int>(min(static_cast<long long>(KB), kb0 + (u1 - u)));
    atomic = true;
    u += kb1 - kb0;
    return true;
  }
};

}  // namespace

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    grad_gemm_kernel(const __grid_constant__ GemmParams p, const __grid_constant__ CUtensorMap mapQ0,
                     const __grid_constant__ CUtensorMap mapX0, const __grid_constant__ CUtensorMap mapQ1,
                     const __grid_constant__ CUtensorMap mapX1, const __grid_constant__ CUtensorMap mapO0,
                     const __grid_constant__ CUtensorMap mapO1) {
  extern __shared__ uint8_t smem_raw[];
  const GSmem L = gcarve(smem_raw);
  const uint32_t warp = threadIdx.x / 32;
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const int pair = blockIdx.x / 2;
  const int n_pairs = gridDim.x / 2;

  // warp roles: epilogue warps first, producer and MMA issuer LAST -- the SMSP arbiter
  // favours the highest warp id, so the single-thread TMA/MMA issue never waits behind
  // the epilogue math.
  constexpr uint32_t kProdWarp = kEpiWarps, kMmaWarp = kEpiWarps + 1;
  if (warp == kProdWarp && lane == 0) {
    tma_prefetch(&mapQ0);
    tma_prefetch(&mapX0);
    if (p.nseg > 1) {
      tma_prefetch(&mapQ1);
      tma_prefetch(&mapX1);
    }
  }
  if (warp == kMmaWarp && lane == 0) {
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
  if (warp == 0) tmem_alloc<2>(L.tmem_ptr, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *L.tmem_ptr;

  if (warp == kProdWarp) {
    // ===================== TMA producer =====================
    {   // whole warp walks the loop, lane 0 issues
      const bool issuer = lane == 0;
      uint32_t stage = 0, phase = 0;
      SegIter iter(p, pair, n_pairs);
      int tile, kb0, kb1;
      bool atomic;
      while (iter.next(tile, kb0, kb1, atomic)) {
        int s, mb, nb;
        tile_decode(p, tile, s, mb, nb);
        const CUtensorMap* mq = s ? &mapQ1 : &mapQ0;
        const CUtensorMap* mx = s ? &mapX1 : &mapX0;
        const int a_row = mb * kPairM + static_cast<int>(rank) * kCtaM;
        const int n0 = nb * kPairN + static_cast<int>(rank) * (kPairN / 2);
        const bool a_mn = p.seg[s].a_mn_major != 0;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&L.empty[stage], phase ^ 1);
          if (p.debug == 2 && kb > kb0 + kStages) {
            if (issuer) {
              if (rank == 0) mbar_arrive(&L.full[stage]);
              else mbar_arrive_cluster(&L.full[stage], 0);
            }
            __syncwarp();
            if (++stage == kStages) { stage = 0; phase ^= 1; }
            continue;
          }
          if (!issuer) {
            __syncwarp();
            if (++stage == kStages) { stage = 0; phase ^= 1; }
            continue;
          }
          if (rank == 0)
            mbar_arrive_expect_tx(&L.full[stage], 2 * (kStageBytesA + kStageBytesB));
          else
            mbar_arrive_cluster(&L.full[stage], 0);
          uint8_t* sa = L.a + stage * kStageBytesA;
          uint8_t* sb = L.b + stage * kStageBytesB;
          if (a_mn) {
            // A = Q^T: two 64(M) x 64(K) swizzle atoms of the row-major Q (K = rows of Q)
            tma_load_2d_pair(mq, &L.full[stage], sa, a_row, kb * kBlockK);
            tma_load_2d_pair(mq, &L.full[stage], sa + kStageBytesA / 2, a_row + 64, kb * kBlockK);
          } else {
            tma_load_2d_pair(mq, &L.full[stage], sa, kb * kBlockK, a_row);
          }
          // MN-major B: two 64(N) x 64(K) swizzle atoms for this CTA's 128 columns of N.
          tma_load_2d_pair(mx, &L.full[stage], sb, n0, kb * kBlockK);
          tma_load_2d_pair(mx, &L.full[stage], sb + kStageBytesB / 2, n0 + 64, kb * kBlockK);
          __syncwarp();
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ===================== MMA issuer (leader CTA, one thread; lean issue loop) =====================
    if (rank == 0) {
      constexpr uint32_t idesc_k = make_idesc_bf16(kPairM, kPairN, 0, 1);
      constexpr uint32_t idesc_mn = make_idesc_bf16(kPairM, kPairN, 1, 1);
      const uint64_t a_desc_k = make_sdesc_sw128(smem_u32(L.a), 0, 1024);
      const uint64_t a_desc_mn = make_sdesc_sw128(smem_u32(L.a), kStageBytesA / 2, 1024);
      // MN-major SW128 B: 16 K rows of 128 B per UMMA_K; LBO = next 64-wide N atom.
      const uint64_t b_desc0 = make_sdesc_sw128(smem_u32(L.b), kStageBytesB / 2, 1024);
      uint32_t stage = 0, phase = 0;
      int it = 0;
      SegIter iter(p, pair, n_pairs);
      int tile, kb0, kb1;
      bool atomic;
      while (iter.next(tile, kb0, kb1, atomic)) {
        int s, mb, nb;
        tile_decode(p, tile, s, mb, nb);
        const bool a_mn = p.seg[s].a_mn_major != 0;
        const uint32_t idesc = a_mn ? idesc_mn : idesc_k;
        const uint64_t a_desc0 = a_mn ? a_desc_mn : a_desc_k;
        const uint32_t a_kstep = a_mn ? (2048 >> 4) : (32 >> 4);   // descriptor units per UMMA_K
        const uint32_t acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&L.tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kPairN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&L.full[stage], phase);
          tc_fence_after();
          if (elect_one()) {
            const uint64_t ad = a_desc0 + static_cast<uint64_t>((stage * kStageBytesA) >> 4);
            const uint64_t bd = b_desc0 + static_cast<uint64_t>((stage * kStageBytesB) >> 4);
            mma_bf16_pair(d_tmem, ad, bd, idesc, kb != kb0);
            mma_bf16_pair(d_tmem, ad + a_kstep, bd + 128, idesc, 1);
            mma_bf16_pair(d_tmem, ad + 2 * a_kstep, bd + 256, idesc, 1);
            mma_bf16_pair(d_tmem, ad + 3 * a_kstep, bd + 384, idesc, 1);
            mma_commit_pair(&L.empty[stage], 0x3);
            if (kb == kb1 - 1) mma_commit_pair(&L.tfull[acc], 0x3);
          }
          __syncwarp();
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        ++it;
      }
    }
  } else {
    // ===================== epilogue =====================
    // Each warp owns 32 rows (its TMEM lane quarter) x 128 columns (its half of N), handled
    // as 4 chunks of 32 columns: TMEM -> registers -> c (acc - r o X_local) -> swizzled smem
    // -> one TMA tile store (whole tiles) or TMA reduce-add (stream-K partial tiles).
    const uint32_t q4 = warp & 3;
    const uint32_t half = warp >> 2;
    uint8_t* stage_out = L.out + warp * kGemmStageOut;
    int it = 0;
    SegIter iter(p, pair, n_pairs);
    int tile, kb0, kb1;
    bool atomic;
    while (iter.next(tile, kb0, kb1, atomic)) {
      int s, mb, nb;
      tile_decode(p, tile, s, mb, nb);
      const GemmSeg& sg = p.seg[s];
      const CUtensorMap* mo = s ? &mapO1 : &mapO0;
      const uint32_t acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int row0 = mb * kPairM + static_cast<int>(rank) * kCtaM + static_cast<int>(q4) * 32;
      const int r_loc = row0 + static_cast<int>(lane);
      const bool row_ok = r_loc < sg.rows;
      const bool with_r = kb0 == 0;   // the -r o X_local term is added exactly once per tile
      const float rr = (row_ok && with_r) ? sg.r[r_loc] : 0.f;
      const __nv_bfloat16* xrow = sg.x + static_cast<size_t>(sg.x_row0 + (row_ok ? r_loc : 0)) * p.d;
      mbar_wait(&L.tfull[acc], acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        const int col0 = nb * kPairN + static_cast<int>(half) * 128 + c * 32;
        const uint32_t taddr = tmem_base + ((q4 * 32u) << 16) + acc * kPairN + half * 128u + c * 32u;
        uint32_t r[32];
        tmem_ld_32x32b_x32(taddr, r);
        tmem_ld_wait();
        if (c == 3) {   // whole accumulator slice read: release it to the MMA warp
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (rank == 0) mbar_arrive(&L.tempty[acc]);
            else mbar_arrive_cluster(&L.tempty[acc], 0);
          }
        }
        if (col0 >= p.d || p.debug != 0) continue;   // warp-uniform
        float v[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) v[k] = p.scale * __uint_as_float(r[k]);
        if (with_r && row_ok) {
          const float cr = p.scale * rr;
          const uint4* xs = reinterpret_cast<const uint4*>(xrow + col0);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            if (col0 + 8 * q >= p.d) break;  // d % 8 == 0: groups of 8 are all-in or all-out
            const uint4 w = __ldg(xs + q);
            const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ww[t]));
              v[q * 8 + 2 * t] = fmaf(-cr, f.x, v[q * 8 + 2 * t]);
              v[q * 8 + 2 * t + 1] = fmaf(-cr, f.y, v[q * 8 + 2 * t + 1]);
            }
          }
        }
        // the previous chunk's bulk store must have finished reading the staging buffer
        if (lane == 0) bulk_wait_read0();
        __syncwarp();
        uint8_t* rowp = stage_out + lane * 128;
#pragma unroll
        for (int u = 0; u < 8; ++u)
          *reinterpret_cast<float4*>(rowp + ((u ^ (lane & 7)) << 4)) =
              make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          if (atomic) tma_reduce_add_2d(mo, stage_out, col0, row0);
          else tma_store_2d(mo, stage_out, col0, row0);
          bulk_commit();
        }
      }
      ++it;
    }
    if (lane == 0) bulk_wait0();
  }

  __syncwarp();   // single-thread producer / MMA roles reconverge before the aligned cluster barrier
  tc_fence_before();
  cluster_sync();
  if (warp == 0) tmem_dealloc<2>(tmem_base, 512);
}

cudaError_t gemm_set_smem() {
  return cudaFuncSetAttribute(grad_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
}

cudaError_t launch_gemm(const GemmParams& p, const CUtensorMap* mapQ, const CUtensorMap* mapX,
                        const CUtensorMap* mapOut, int grid, cudaStream_t s) {
  const CUtensorMap& q1 = p.nseg > 1 ? mapQ[1] : mapQ[0];
  const CUtensorMap& x1 = p.nseg > 1 ? mapX[1] : mapX[0];
  const CUtensorMap& o1 = p.nseg > 1 ? mapOut[1] : mapOut[0];
  if (grid < 2) grid = 2;
  grid &= ~1;
  grad_gemm_kernel<<<grid, kThreads, kSmemBytes, s>>>(p, mapQ[0], mapX[0], q1, x1, mapOut[0], o1);
  return cudaGetLastError();
}

}  // namespace fc
