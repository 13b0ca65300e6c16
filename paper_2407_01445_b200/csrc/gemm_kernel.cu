// gemm_kernel.cu -- weighted-gradient GEMM (FastCLIP pass 2b) for sm_100a.
//
//   dE1[L] = c (Q'_R  E2[G] - r o E2[L]),   dE2[L] = c (Q'_C  E1[G] - r o E1[L])
// (engine.cpp:77-121 regrouped: Q[i,j] = P1[i,j] + P2[j,i], r_i = a_i S1_i + b_i S2_i,
//  c = 1/(Bl (B-1))). A = Q' (bf16, K-major; at K = 1 the dE2 GEMM reads Q^T through an
// MN-major A operand), B = E (bf16, N = d contiguous => MN-major UMMA operand), fp32
// accumulation in TMEM.
//
// The GEMM is skinny (N = d = 512, K = B = 5120) and both operands stream, so its limit is
// the L2 -> SM operand bandwidth: each CTA pair (cta_group::2) owns a 256 x 512 tile -- two
// N = 256 accumulators that fill TMEM and share every A k-block (48 KB per 1024 MMA cycles
// per CTA). Schedule: stream-K over (tile, k-block) -- every pair runs the same number of
// k-blocks (+-1); partial tiles are reduced with TMA reduce-add into the gradient rows, which
// a side-branch kernel zeroed earlier in the step; the unit holding k-block 0 of a tile also
// adds the local term -c r o E_L.
//
#include "kernels.cuh"
#include "sm100.cuh"

namespace fc {

namespace {

struct GSmem {
  uint8_t* a;     // kGemmStages x 16 KB (own 128 rows x 64 k)
  uint8_t* b;     // kGemmStages x 32 KB (own 128 columns of each N half x 64 k)
  uint8_t* out;   // kGemmEpiWarps x 4 KB epilogue staging (TMA reduce-add source)
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
  L.b = p + kGemmStages * kStageBytesA;
  L.out = L.b + kGemmStages * kGemmStageBytesB;
  uint64_t* bars = reinterpret_cast<uint64_t*>(L.out + kGemmEpiWarps * kGemmStageOut);
  L.full = bars;
  L.empty = bars + kGemmStages;
  L.tfull = bars + 2 * kGemmStages;
  L.tempty = bars + 2 * kGemmStages + 1;
  L.tmem_ptr = reinterpret_cast<uint32_t*>(bars + 2 * kGemmStages + 2);
  return L;
}

// pair tile -> (segment, row block of 256 rows, column block of 512)
__device__ __forceinline__ void tile_decode(const GemmParams& p, int t, int& s, int& mb, int& nb) {
  const int per_seg0 = p.n_mb[0] * p.n_nb;
  s = t < per_seg0 ? 0 : 1;
  const int local = t - (s ? per_seg0 : 0);
  nb = local % p.n_nb;
  mb = local / p.n_nb;
}

// The pair's stream-K work: contiguous range of (tile, k-block) units.
struct UnitIter {
  int KB;
  long long u, u1;
  __device__ UnitIter(const GemmParams& p, int pair) {
    KB = p.kb_total;
    u = p.unit_lo[pair];
    u1 = p.unit_lo[pair + 1];
  }
  __device__ bool next(int& tile, int& kb0, int& kb1) {
    if (u >= u1) return false;
    tile = static_cast<int>(u / KB);
    kb0 = static_cast<int>(u % KB);
    kb1 = static_cast<int>(min(static_cast<long long>(KB), kb0 + (u1 - u)));
    u += kb1 - kb0;
    return true;
  }
};

}  // namespace

__global__ void __launch_bounds__(kGemmThreads, 1)
    grad_gemm_kernel(const __grid_constant__ GemmParams p, const __grid_constant__ CUtensorMap mapQ0,
                     const __grid_constant__ CUtensorMap mapX0, const __grid_constant__ CUtensorMap mapQ1,
                     const __grid_constant__ CUtensorMap mapX1, const __grid_constant__ CUtensorMap mapO0,
                     const __grid_constant__ CUtensorMap mapO1) {
  extern __shared__ uint8_t smem_raw[];
#ifdef FC_PROFILE
  long long g_entry;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_entry));
#endif
  const GSmem L = gcarve(smem_raw);
  griddep_launch_dependents();
  const uint32_t warp = threadIdx.x / 32;
  const uint32_t lane = lane_id();
  const uint32_t prank = cluster_ctarank();          // rank inside the CTA pair
  const int pair = blockIdx.x / 2;
  constexpr uint16_t kPairMask = 0x3;

  constexpr uint32_t kProdWarp = kGemmEpiWarps, kMmaWarp = kGemmEpiWarps + 1;
  if (warp == kProdWarp && lane == 0) {
    tma_prefetch(&mapQ0);
    tma_prefetch(&mapX0);
    if (p.nseg > 1) {
      tma_prefetch(&mapQ1);
      tma_prefetch(&mapX1);
    }
  }
  if (warp == kMmaWarp && lane == 0) {
    for (int i = 0; i < kGemmStages; ++i) {
      mbar_init(&L.full[i], 2);           // both producers of the pair (leader's barrier is used)
      mbar_init(&L.empty[i], 1);          // MMA commit (multicast to both CTAs)
    }
    mbar_init(&L.tfull[0], 1);
    mbar_init(&L.tempty[0], 2 * kGemmEpiWarps);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<2>(L.tmem_ptr, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *L.tmem_ptr;

  if (warp == kProdWarp) {
    // ===================== TMA producer (whole warp walks, lane 0 issues) =====================
    const bool issuer = lane == 0;
    uint32_t stage = 0, phase = 0;
    griddep_wait();   // Q' / X come from the preceding kernels (barrier init / TMEM alloc overlapped them)
    UnitIter iter(p, pair);
    int tile, kb0, kb1;
    while (iter.next(tile, kb0, kb1)) {
      int s, mb, nb;
      tile_decode(p, tile, s, mb, nb);
      const CUtensorMap* mq = s ? &mapQ1 : &mapQ0;
      const CUtensorMap* mx = s ? &mapX1 : &mapX0;
      const int a_row = mb * kPairM + static_cast<int>(prank) * kCtaM;
      const int n_blk = nb * kGemmN;
      const bool a_mn = p.seg[s].a_mn_major != 0;
      const bool half1 = n_blk + kPairN < p.d;   // this block's second N half has columns
      const uint32_t b_bytes = 2 * (half1 ? 2 : 1) * kStageBytesB;
      for (int kb = kb0; kb < kb1; ++kb) {
        mbar_wait(&L.empty[stage], phase ^ 1);
        if (issuer) {
          uint8_t* sa = L.a + stage * kStageBytesA;
          uint8_t* sb = L.b + stage * kGemmStageBytesB;
          const int k0 = kb * kBlockK;
          if (prank == 0) mbar_arrive_expect_tx(&L.full[stage], b_bytes + 2 * kStageBytesA);
          else mbar_arrive_cluster(&L.full[stage], 0);
          if (a_mn) {
            // A = Q^T: two 64(M) x 64(K) swizzle atoms of the row-major Q (K = rows of Q)
            tma_load_2d_pair(mq, &L.full[stage], sa, a_row, k0);
            tma_load_2d_pair(mq, &L.full[stage], sa + kStageBytesA / 2, a_row + 64, k0);
          } else {
            tma_load_2d_pair(mq, &L.full[stage], sa, k0, a_row);
          }
          // B slab h of this CTA: columns n_blk + h*256 + prank*128 .. +128 (two 64-wide atoms)
          for (int h = 0; h < (half1 ? 2 : 1); ++h) {
            const int n0 = n_blk + h * kPairN + static_cast<int>(prank) * (kPairN / 2);
            uint8_t* dst = sb + h * kStageBytesB;
            tma_load_2d_pair(mx, &L.full[stage], dst, n0, k0 + p.seg[s].x_krow0);
            tma_load_2d_pair(mx, &L.full[stage], dst + kStageBytesB / 2, n0 + 64, k0 + p.seg[s].x_krow0);
          }
        }
        __syncwarp();
        if (++stage == kGemmStages) { stage = 0; phase ^= 1; }
      }
    }
  } else if (warp == kMmaWarp) {
    // ===================== MMA issuer (pair leader; whole warp in the loop, one lane issues) =====================
    if (prank == 0) {
      constexpr uint32_t idesc_k = make_idesc_bf16(kPairM, kPairN, 0, 1);
      constexpr uint32_t idesc_mn = make_idesc_bf16(kPairM, kPairN, 1, 1);
      const uint64_t a_desc_k = make_sdesc_sw128(smem_u32(L.a), 0, 1024);
      const uint64_t a_desc_mn = make_sdesc_sw128(smem_u32(L.a), kStageBytesA / 2, 1024);
      // MN-major SW128 B: 16 K rows of 128 B per UMMA_K; LBO = next 64-wide N atom.
      const uint64_t b_desc0 = make_sdesc_sw128(smem_u32(L.b), kStageBytesB / 2, 1024);
      constexpr uint32_t kBHalf = kStageBytesB >> 4;   // descriptor offset of N half 1
      uint32_t stage = 0, phase = 0;
      int it = 0;
#ifdef FC_PROFILE
      long long c0 = clock64(), c_tempty = 0, c_full = 0, c_first = -1;
#endif
      UnitIter iter(p, pair);
      int tile, kb0, kb1;
      while (iter.next(tile, kb0, kb1)) {
        int s, mb, nb;
        tile_decode(p, tile, s, mb, nb);
        const bool a_mn = p.seg[s].a_mn_major != 0;
        const bool half1 = nb * kGemmN + kPairN < p.d;
        const uint32_t idesc = a_mn ? idesc_mn : idesc_k;
        const uint64_t a_desc0 = a_mn ? a_desc_mn : a_desc_k;
        const uint32_t a_kstep = a_mn ? (2048 >> 4) : (32 >> 4);   // descriptor units per UMMA_K
#ifdef FC_PROFILE
        long long t0 = clock64();
#endif
        mbar_wait(&L.tempty[0], (it & 1) ^ 1);   // the epilogue drained the previous unit
#ifdef FC_PROFILE
        c_tempty += clock64() - t0;
#endif
        tc_fence_after();
        for (int kb = kb0; kb < kb1; ++kb) {
#ifdef FC_PROFILE
          long long t1 = clock64();
#endif
          mbar_wait(&L.full[stage], phase);
#ifdef FC_PROFILE
          c_full += clock64() - t1;
          if (c_first < 0) c_first = clock64() - c0;
#endif
          tc_fence_after();
          if (elect_one()) {
            const uint64_t ad = a_desc0 + static_cast<uint64_t>((stage * kStageBytesA) >> 4);
            const uint64_t bd = b_desc0 + static_cast<uint64_t>((stage * kGemmStageBytesB) >> 4);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint32_t accum = (kb != kb0 || k != 0) ? 1u : 0u;
              mma_bf16_pair(tmem_base, ad + k * a_kstep, bd + 128 * k, idesc, accum);
              if (half1) mma_bf16_pair(tmem_base + kPairN, ad + k * a_kstep, bd + kBHalf + 128 * k, idesc, accum);
            }
            mma_commit_pair(&L.empty[stage], kPairMask);
            if (kb == kb1 - 1) mma_commit_pair(&L.tfull[0], kPairMask);
          }
          __syncwarp();
          if (++stage == kGemmStages) { stage = 0; phase ^= 1; }
        }
        ++it;
      }
#ifdef FC_PROFILE
      if (lane == 0 && p.dbg_out) {
        long long* o = p.dbg_out + blockIdx.x * 16;
        o[0] = clock64() - c0; o[1] = c_tempty; o[2] = c_full; o[3] = c_first; o[4] = it;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(o[5]));
      }
#endif
    }
  } else if (warp < kGemmEpiWarps) {
    // ===================== epilogue =====================
    // Warp w owns 32 rows (TMEM lane quarter w & 3) x 256 columns (N half w >> 2) of the
    // pair's 256 x 512 accumulator: 8 chunks of 32 columns, TMEM -> registers ->
    // c (acc - r o X_L) -> swizzled smem -> TMA reduce-add into the zeroed gradient rows.
    constexpr int kEpiCols = kGemmN / (kGemmEpiWarps / 4);   // columns per warp
    constexpr int kChunks = kEpiCols / 32;
    const uint32_t q4 = warp & 3;
    const uint32_t cg = warp >> 2;
    uint8_t* stage_out = L.out + warp * kGemmStageOut;
    // r_i (per-anchor kernel) and the X rows are read before the first accumulator wait:
    // wait for the predecessor grid like the producer does (programmatic launch)
    griddep_wait();
#ifdef FC_PROFILE
    long long e0 = clock64(), e_wait = 0;
#endif
    int it = 0;
    UnitIter iter(p, pair);
    int tile, kb0, kb1;
    while (iter.next(tile, kb0, kb1)) {
      int s, mb, nb;
      tile_decode(p, tile, s, mb, nb);
      const GemmSeg& sg = p.seg[s];
      const CUtensorMap* mo = s ? &mapO1 : &mapO0;
      const int row0 = mb * kPairM + static_cast<int>(prank) * kCtaM + static_cast<int>(q4) * 32;
      const int r_loc = row0 + static_cast<int>(lane);
      const bool row_ok = r_loc < sg.rows;
      // the unit holding k-block 0 adds the local term -c r o X_L exactly once per tile; its X
      // loads are software-pipelined one chunk ahead (the first before the accumulator wait)
      const bool with_r = kb0 == 0 && sg.r != nullptr;
      const float cr = (row_ok && with_r) ? p.scale * sg.r[r_loc] : 0.f;
      const uint4* xrow = reinterpret_cast<const uint4*>(sg.x + static_cast<size_t>(sg.x_row0 + (row_ok ? r_loc : 0)) * p.d);
      uint4 xn[4];
      auto load_x = [&](int cc) {
        const int col0 = nb * kGemmN + static_cast<int>(cg) * kEpiCols + cc * 32;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          xn[q] = (with_r && row_ok && col0 + 8 * q < p.d) ? __ldg(xrow + col0 / 8 + q) : make_uint4(0u, 0u, 0u, 0u);
      };
      load_x(0);
#ifdef FC_PROFILE
      long long t0 = clock64();
#endif
      mbar_wait(&L.tfull[0], it & 1);
#ifdef FC_PROFILE
      e_wait += clock64() - t0;
#endif
      tc_fence_after();
#pragma unroll 1
      for (int cc = 0; cc < kChunks; ++cc) {
        const int tcol = static_cast<int>(cg) * kEpiCols + cc * 32;   // column inside the 512-wide block
        const int col0 = nb * kGemmN + tcol;
        const bool live = col0 < p.d && row0 < sg.rows;          // warp-uniform
        uint32_t r[32];
        if (live || cc == kChunks - 1) {
          tmem_ld_32x32b_x32(tmem_base + ((q4 * 32u) << 16) + static_cast<uint32_t>(tcol), r);
          tmem_ld_wait();
        }
        if (cc == kChunks - 1) {   // this warp's accumulator slice is in registers: release it
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (prank == 0) mbar_arrive(&L.tempty[0]);
            else mbar_arrive_cluster(&L.tempty[0], 0);
          }
        }
        if (!live) continue;
        float v[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) v[k] = p.scale * __uint_as_float(r[k]);
        if (with_r) {
          uint4 xc[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) xc[q] = xn[q];
          if (cc + 1 < kChunks) load_x(cc + 1);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t ww[4] = {xc[q].x, xc[q].y, xc[q].z, xc[q].w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ww[u]));
              v[q * 8 + 2 * u] = fmaf(-cr, f.x, v[q * 8 + 2 * u]);
              v[q * 8 + 2 * u + 1] = fmaf(-cr, f.y, v[q * 8 + 2 * u + 1]);
            }
          }
        }
        // the previous chunk's bulk reduce must have finished reading the staging buffer
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
          tma_reduce_add_2d(mo, stage_out, col0, row0);
          bulk_commit();
        }
      }
      ++it;
    }
    if (lane == 0) bulk_wait0();
#ifdef FC_PROFILE
    if (warp == 0 && lane == 0 && p.dbg_out) {
      long long* o = p.dbg_out + blockIdx.x * 16 + 8;
      o[0] = clock64() - e0; o[1] = e_wait;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(o[2]));
      o[3] = g_entry;
    }
#endif
  }

  __syncwarp();   // single-lane producer / MMA roles reconverge before the aligned cluster barrier
  tc_fence_before();
  cluster_sync();
  if (warp == 0) tmem_dealloc<2>(tmem_base, 512);
  // every CTA is past its producer's griddep_wait here, so pass 2 (the last reader of the
  // bounds) has completed
  if (blockIdx.x == 0 && static_cast<int>(threadIdx.x) < 4 * p.n_reset && p.reset_at_exit) p.reset_at_exit[threadIdx.x] = 0.f;
}

cudaError_t launch_gemm(bool pdl, const GemmParams& p, const CUtensorMap* mapQ, const CUtensorMap* mapX,
                          const CUtensorMap* mapOut, int grid, cudaStream_t s) {
  const CUtensorMap& q1 = p.nseg > 1 ? mapQ[1] : mapQ[0];
  const CUtensorMap& x1 = p.nseg > 1 ? mapX[1] : mapX[0];
  const CUtensorMap& o1 = p.nseg > 1 ? mapOut[1] : mapOut[0];
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(kGemmThreads, 1, 1);
  cfg.dynamicSmemBytes = kGemmSmemBytes;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, grad_gemm_kernel, p, mapQ[0], mapX[0], q1, x1, mapOut[0], o1);
}

cudaError_t gemm_set_smem() {
  return cudaFuncSetAttribute(grad_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kGemmSmemBytes);
}

}  // namespace fc
