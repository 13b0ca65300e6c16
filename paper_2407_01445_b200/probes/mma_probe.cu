// mma_probe.cu -- microbenchmark of the tcgen05 issue rate (diagnostics only, NOT part of the
// product library; build it on its own:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -shared \
//        -I paper_2407_01445_b200/csrc paper_2407_01445_b200/probes/mma_probe.cu -o /tmp/libmma_probe.so
// and call probe_mma / probe_ring through ctypes; scripts/mma_probe2.py): one CTA pair issues n back-to-back bf16 MMAs on resident shared-memory
// operands (M = 256 pair, N = 256, K = 16 each), optionally committing every `commit_every`
// MMAs to an mbarrier; the leader reports elapsed SM cycles.
#include "kernels.cuh"
#include "sm100.cuh"

namespace fc {
cudaError_t launch_ring_probe(int n_pairs, int n_kb, int tile_kb, int epi, long long* cycles, cudaStream_t s);
cudaError_t launch_mma_probe(int n_pairs, int n_mma, int commit_every, long long* cycles, cudaStream_t s);
}  // namespace fc

namespace fc {

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    mma_probe_kernel(int n_mma, int commit_every, long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + 64 * 1024);
  uint32_t* tptr = reinterpret_cast<uint32_t*>(bar + 2);
  const uint32_t warp = threadIdx.x / 32;
  const uint32_t rank = cluster_ctarank();
  // zero operands (values do not matter for the rate)
  // bf16 operands in [0.5, 1) with varying mantissas (random-like bit patterns, finite values)
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) {
    uint32_t h = (i * 2654435761u) ^ (blockIdx.x * 40503u);
    reinterpret_cast<uint32_t*>(base)[i] = 0x3F003F00u | (h & 0x007F007Fu) | ((h >> 8) & 0x80008000u);
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) tmem_alloc<2>(tptr, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tptr;
  if (warp == 1 && rank == 0) {
    constexpr uint32_t idesc = make_idesc_bf16(kPairM, kPairN, 0, 0);
    const uint32_t a0 = smem_u32(base);
    const uint32_t b0 = smem_u32(base + 32 * 1024);
    uint32_t ph = 0;
    long long t0 = clock64();
    if (lane_id() == 0) {
      if (commit_every <= 0) {
        for (int i = 0; i < n_mma; ++i) {
          const int k = i & 3;
          mma_bf16_pair(tmem + (i & 1) * 256, make_sdesc_sw128(a0 + k * 32, 0, 1024),
                        make_sdesc_sw128(b0 + k * 32, 0, 1024), idesc, 1);
        }
      } else {
        // realistic k-block loop: 4 MMAs per block with precomputed descriptors;
        // commit_every bit0: try_wait on a completed barrier, bit1: fence, bit2: commit,
        // bit3: MN-major B operand, bit4: MN-major A operand (operand-major rate check)
        const bool bmn = commit_every & 8, amn = commit_every & 16;
        const uint32_t idesc2 = amn ? (bmn ? make_idesc_bf16(kPairM, kPairN, 1, 1) : make_idesc_bf16(kPairM, kPairN, 1, 0))
                                    : (bmn ? make_idesc_bf16(kPairM, kPairN, 0, 1) : idesc);
        const uint64_t ad0 = make_sdesc_sw128(a0, amn ? 8192 : 0, 1024), bd0 = make_sdesc_sw128(b0, bmn ? 8192 : 0, 1024);
        const uint32_t ak = amn ? 128 : 2, bk = bmn ? 128 : 2;
        mbar_arrive(&bar[0]);   // complete phase 0 so waits on parity 0 return at once
        for (int i = 0; i < n_mma / 4; ++i) {
          if (commit_every & 1) mbar_wait(&bar[0], 0);
          if (commit_every & 2) tc_fence_after();
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma_bf16_pair(tmem + (i & 1) * 256, ad0 + ak * k, bd0 + bk * k, idesc2, 1);
          if (commit_every & 4) mma_commit_pair(&bar[0] + 0, 0x1);
        }
      }
      mma_commit_pair(&bar[1], 0x1);
    }
    __syncwarp();
    mbar_wait(&bar[1], ph);
    long long t1 = clock64();
    if (threadIdx.x == 32) cycles[blockIdx.x / 2] = t1 - t0;
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 0) tmem_dealloc<2>(tmem, 512);
}

// Ring protocol probe: producer warp (both CTAs) waits empty[s], arrives on the leader's
// full[s] (peer: remote arrive); the leader's MMA warp waits full[s], issues 4 MMAs, commits
// empty[s] to both CTAs -- the exact handshake of the loss-step kernels, minus the TMA data.
// Every `tile_kb` k blocks the accumulator buffer flips and (if epi) an epilogue warp round
// trip through tfull/tempty is made.
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(640, 1)
    ring_probe_kernel(int n_kb, int tile_kb, int epi, long long* cycles) {
  const int n_epi = 1 + (blockDim.x - 128) / 32;   // warp 1 + warps >= 4
  constexpr int S = 5;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(base + 64 * 1024);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tptr = reinterpret_cast<uint32_t*>(tempty + 2);
  const uint32_t warp = threadIdx.x / 32;
  const uint32_t rank = cluster_ctarank();
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0x3F803F80u;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) { mbar_init(&full[i], 2); mbar_init(&empty[i], 1); }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 2 * n_epi); }
    fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) tmem_alloc<2>(tptr, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = *tptr;
  const int n_tiles = n_kb / tile_kb;
  long long t0 = clock64();
  if (warp == 3) {   // producer
    uint32_t st = 0, ph = 0;
    for (int i = 0; i < n_kb; ++i) {
      mbar_wait(&empty[st], ph ^ 1);
      if (elect_one()) {
        if (rank == 0) mbar_arrive(&full[st]);
        else mbar_arrive_cluster(&full[st], 0);
      }
      __syncwarp();
      if (++st == S) { st = 0; ph ^= 1; }
    }
  } else if (warp == 2 && rank == 0) {   // MMA
    constexpr uint32_t idesc = make_idesc_bf16(kPairM, kPairN, 0, 0);
    const uint64_t ad0 = make_sdesc_sw128(smem_u32(base), 0, 1024), bd0 = make_sdesc_sw128(smem_u32(base + 32768), 0, 1024);
    uint32_t st = 0, ph = 0;
    for (int t = 0; t < n_tiles; ++t) {
      const uint32_t acc = t & 1;
      if (epi) { mbar_wait(&tempty[acc], ((t >> 1) & 1) ^ 1); tc_fence_after(); }
      for (int kb = 0; kb < tile_kb; ++kb) {
        mbar_wait(&full[st], ph);
        tc_fence_after();
        if (elect_one()) {
          const uint64_t ad = ad0 + ((st * 4096) >> 4), bd = bd0 + ((st * 4096) >> 4);
          mma_bf16_pair(tmem + acc * 256, ad, bd, idesc, kb != 0);
          mma_bf16_pair(tmem + acc * 256, ad + 2, bd + 2, idesc, 1);
          mma_bf16_pair(tmem + acc * 256, ad + 4, bd + 4, idesc, 1);
          mma_bf16_pair(tmem + acc * 256, ad + 6, bd + 6, idesc, 1);
          mma_commit_pair(&empty[st], 0x3);
          if (epi && kb == tile_kb - 1) mma_commit_pair(&tfull[acc], 0x3);
        }
        __syncwarp();
        if (++st == S) { st = 0; ph ^= 1; }
      }
    }
  } else if ((warp == 1 || warp >= 4) && epi) {   // epilogue stand-ins (both CTAs)
    for (int t = 0; t < n_tiles; ++t) {
      const uint32_t acc = t & 1;
      mbar_wait(&tfull[acc], (t >> 1) & 1);
      tc_fence_after();
      uint32_t r[32];
      tmem_ld_32x32b_x32(tmem + (((warp & 3) * 32u) << 16) + acc * 256, r);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) {
        if (rank == 0) mbar_arrive(&tempty[acc]);
        else mbar_arrive_cluster(&tempty[acc], 0);
      }
      if (r[0] == 0x12345678u) cycles[0] = 0;
    }
  }
  __syncwarp();
  tc_fence_before();
  cluster_sync();
  long long t1 = clock64();
  if (threadIdx.x == 0 && rank == 0) cycles[blockIdx.x / 2] = t1 - t0;
  if (warp == 0) tmem_dealloc<2>(tmem, 512);
}

cudaError_t launch_ring_probe(int n_pairs, int n_kb, int tile_kb, int epi, long long* cycles, cudaStream_t s) {
  const int smem = 64 * 1024 + 2048;
  cudaError_t e = cudaFuncSetAttribute(ring_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  ring_probe_kernel<<<n_pairs * 2, 128 + 32 * (epi > 1 ? epi - 1 : 0), smem, s>>>(n_kb, tile_kb, epi, cycles);
  return cudaGetLastError();
}

cudaError_t launch_mma_probe(int n_pairs, int n_mma, int commit_every, long long* cycles, cudaStream_t s) {
  const int smem = 64 * 1024 + 2048;
  cudaError_t e = cudaFuncSetAttribute(mma_probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  mma_probe_kernel<<<n_pairs * 2, 128, smem, s>>>(n_mma, commit_every, cycles);
  return cudaGetLastError();
}

}  // namespace fc

extern "C" int probe_mma(int n_pairs, int n_mma, int commit_every, long long* cycles, void* stream) {
  return static_cast<int>(fc::launch_mma_probe(n_pairs, n_mma, commit_every, cycles, static_cast<cudaStream_t>(stream)));
}
extern "C" int probe_ring(int n_pairs, int n_kb, int tile_kb, int epi, long long* cycles, void* stream) {
  return static_cast<int>(fc::launch_ring_probe(n_pairs, n_kb, tile_kb, epi, cycles, static_cast<cudaStream_t>(stream)));
}
