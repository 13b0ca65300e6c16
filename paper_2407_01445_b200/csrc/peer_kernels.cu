// peer_kernels.cu -- NVLink peer-memory all-gather for the K > 1 step (trainer.cpp:422-425
// "feature-gather" and :459-487 u/tau gathers).
//
// Every rank maps the gather destinations of all ranks (CUDA IPC, handles exchanged once over
// NCCL at creation). One kernel per gather: its CTAs store this rank's slice straight into
// every rank's destination buffer over NVLink (16-byte stores, grid-strided), the last CTA to
// finish (device-scope ticket) publishes a per-step sequence number into each peer's flag slot
// for this rank (one system-scope release fence, then relaxed flag stores back to back) and
// then waits until every rank's flag in the LOCAL flag array carries the same sequence number
// (relaxed polling, then a system-scope acquire fence). The kernel therefore
// completes only when the whole gathered buffer is in local HBM -- a stream-ordered all-gather
// with no NCCL launch and no proxy thread (~20-30 us per NCCL gather on this system vs a few
// microseconds of NVLink traffic for the payload and ~2.6 MB embedding slices). With the
// overlapped step (loss_step.cu) the gathers run on their own stream and the passes that read
// their data poll the same flags inside their grids; those launches use the lean variant below,
// whose CTAs fit beside a similarity-pass CTA.
#include <cstdint>

#include <cuda_runtime.h>

#include "kernels.cuh"

namespace fc {

namespace {

__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// release/acquire fence at system scope: orders this thread's (and, cumulatively, the CTA's
// barrier-ordered) prior stores before its later ones for every observer, without the
// sequential-consistency cost of fence.sc.sys (__threadfence_system)
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

}  // namespace

__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

constexpr int kErrCollectiveAborted = 8;   // FC_ERR_COLLECTIVE_ABORTED (CollectiveAborted, errors.hpp)

constexpr uint32_t kBulkChunk = 16384;   // bytes per bulk chunk (two chunks of shared staging per CTA)

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Bulk-copy engine path: thread 0 of each CTA streams its chunks of the slices through two
// shared-memory buffers -- one bulk load from local memory, then one bulk store per rank into
// the peer-mapped destination (the copy engine issues the NVLink writes instead of 16-byte LSU
// stores from every thread) -- and waits for the stores' completion before the grid ticket.
__device__ void gather_bulk(const PeerGather& g, uint8_t* stage, uint64_t* bar) {
  if (threadIdx.x != 0) return;
  for (int b = 0; b < 2; ++b)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar + b)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  uint32_t it = 0;
  for (int t = 0; t < g.n_src; ++t) {
    if (t == g.wait_src) asm volatile("griddepcontrol.wait;" ::: "memory");   // the predecessor's outputs
    const size_t bytes = g.bytes[t];
    for (size_t off = static_cast<size_t>(blockIdx.x) * kBulkChunk; off < bytes;
         off += static_cast<size_t>(gridDim.x) * kBulkChunk, ++it) {
      const uint32_t sz = static_cast<uint32_t>(bytes - off < kBulkChunk ? bytes - off : kBulkChunk);
      const uint32_t b = it & 1;
      uint8_t* buf = stage + b * kBulkChunk;
      // the stores that read this buffer two chunks ago are done reading it
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar + b)), "r"(sz) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       smem_addr(buf)),
                   "l"(reinterpret_cast<uint64_t>(g.src[t] + off)), "r"(sz), "r"(smem_addr(bar + b))
                   : "memory");
      asm volatile(
          "{\n\t.reg .pred P1;\n\t"
          "WAIT_%=:\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
          "@P1 bra DONE_%=;\n\t"
          "bra WAIT_%=;\n\t"
          "DONE_%=:\n\t}" ::"r"(smem_addr(bar + b)),
          "r"((it >> 1) & 1u)
          : "memory");
      for (int k = 0; k < g.world; ++k)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                         reinterpret_cast<uint64_t>(g.dst[t][k] + static_cast<size_t>(g.rank) * bytes + off)),
                     "r"(smem_addr(buf)), "r"(sz)
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");   // every store performed
  asm volatile("fence.proxy.async.global;" ::: "memory");     // async-proxy writes -> generic observers
}

// Sources [t0, t1) as one concatenated index space of 16-byte chunks, grid-strided, kU
// independent loads in flight per thread before the stores to every rank.
template <int kU>
__device__ void gather_lsu(const PeerGather& g, int t0, int t1) {
  size_t total = 0;
  for (int t = t0; t < t1; ++t) total += g.bytes[t] / 16;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  for (size_t i0 = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i0 < total; i0 += kU * stride) {
    uint4 v[kU];
    int ts[kU];
    size_t js[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      size_t j = i0 + u * stride;
      int t = t0;
      ts[u] = -1;
      if (j < total) {
        while (j >= g.bytes[t] / 16) {
          j -= g.bytes[t] / 16;
          ++t;
        }
        ts[u] = t;
        js[u] = j;
        v[u] = reinterpret_cast<const uint4*>(g.src[t])[j];
      }
    }
#pragma unroll 1
    for (int k = 0; k < g.world; ++k) {
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (ts[u] >= 0)
          reinterpret_cast<uint4*>(g.dst[ts[u]][k] + static_cast<size_t>(g.rank) * g.bytes[ts[u]])[js[u]] = v[u];
    }
  }
}

// Two equal-size sources (the embedding slices), lean CTAs: chunk i of both and chunk i + stride
// of both -- four 16-byte loads in flight per thread within the 32-register budget.
__device__ void gather_pair_lean(const PeerGather& g) {
  const size_t n = g.bytes[0] / 16;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  const uint4* a = reinterpret_cast<const uint4*>(g.src[0]);
  const uint4* b = reinterpret_cast<const uint4*>(g.src[1]);
  const size_t off = static_cast<size_t>(g.rank) * g.bytes[0];
  for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += 2 * stride) {
    const size_t j = i + stride < n ? i + stride : i;   // past the end: chunk i twice (same bytes)
    const uint4 a0 = a[i], b0 = b[i], a1 = a[j], b1 = b[j];
#pragma unroll 1
    for (int k = 0; k < g.world; ++k) {
      uint4* da = reinterpret_cast<uint4*>(g.dst[0][k] + off);
      uint4* db = reinterpret_cast<uint4*>(g.dst[1][k] + off);
      da[i] = a0;
      db[i] = b0;
      da[j] = a1;
      db[j] = b1;
    }
  }
}

// kLean: a gather that runs beside pass 1 / pass 2 (whose producers wait for its flags), so one
// of its CTAs must fit next to a similarity-pass CTA: 128 threads at <= 32 registers (1024 per
// warp -- what the pass CTA's 96-register warps leave free on its two fuller SM sub-partitions);
// the embedding slices with four loads in flight per thread, the payload's small sources with
// one. Otherwise up to 256 threads, four loads in flight.
template <bool kLean>
__global__ void __launch_bounds__(kLean ? 128 : 256, kLean ? 16 : 1) peer_gather_kernel(PeerGather g) {
  constexpr int kU = 4;
  if (kProfStamps && g.dbg && blockIdx.x == 0 && threadIdx.x == 0) g.dbg[0] = gtimer();
  if (g.early_trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // ---- this rank's slices -> every rank's destination (row offset rank * bytes) ----
  extern __shared__ __align__(128) uint8_t bulk_stage[];
  if (!kLean && g.bulk) gather_bulk(g, bulk_stage, reinterpret_cast<uint64_t*>(bulk_stage + 2 * kBulkChunk));
  if (kLean && g.n_src == 2 && g.bytes[0] == g.bytes[1] && g.wait_src < 0) {
    gather_pair_lean(g);   // the embedding slices
  } else if (kLean) {
    gather_lsu<1>(g, 0, g.n_src);   // the payload (no programmatic predecessor on the lean path)
  } else if (!g.bulk) {
    // the sources written before this kernel started, then (after griddepcontrol.wait) the ones
    // its predecessor writes: each range is one flattened index space of 16-byte chunks, so a
    // thread keeps four loads in flight across small sources too (one round trip per batch,
    // not one per source)
    const int w = (g.wait_src >= 0 && g.wait_src < g.n_src) ? g.wait_src : g.n_src;
    gather_lsu<kU>(g, 0, w);
    if (w < g.n_src) {
      asm volatile("griddepcontrol.wait;" ::: "memory");   // the predecessor's outputs
      gather_lsu<kU>(g, w, g.n_src);
    }
  }
  // ---- grid completion: the last CTA publishes and waits ----
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_acq_rel_sys();      // this CTA's peer stores (ordered by the barrier) before the ticket
    const unsigned ticket = atomicAdd(g.ticket, 1u);
    last = ticket == gridDim.x - 1;
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  *g.ticket = 0u;             // re-arm for the next gather (stream order)
  if (kProfStamps && g.dbg) g.dbg[1] = gtimer();
  // one release fence orders every CTA's stores (acquired through the ticket) before all the
  // flag stores, which then go out back to back (a release per store would serialise them
  // behind one NVLink round trip each)
  fence_acq_rel_sys();
  for (int k = 0; k < g.world; ++k) st_relaxed_sys(g.peer_flag[k] + g.rank, g.seq);
  if (kProfStamps && g.dbg) g.dbg[2] = gtimer();
  // wait for every rank's slice. A peer that stopped stepping is detected after timeout_ns: this
  // rank then poisons every rank (fabric.cpp:228-235); a poisoned rank stops waiting at once.
  const long long t0 = gtimer();
  for (int k = 0; k < g.world; ++k) {
    unsigned spins = 0;
    while (ld_relaxed_sys(g.my_flag + k) < g.seq) {
      __nanosleep(64);
      if ((++spins & 255u) != 0u) continue;   // the abort word and the clock: every 256 polls
      if (ld_relaxed_sys(g.my_abort) != 0ull) {   // a peer gave up on this collective
        atomicCAS(g.err, 0, kErrCollectiveAborted);
        return;
      }
      if (gtimer() - t0 > g.timeout_ns) {
        for (int j = 0; j < g.world; ++j) st_relaxed_sys(g.peer_abort[j], g.seq);
        atomicCAS(g.err, 0, kErrCollectiveAborted);
        return;
      }
    }
  }
  fence_acq_rel_sys();        // acquire: the peers' slices are read only after their flags
  if (kProfStamps && g.dbg) g.dbg[3] = gtimer();
}

cudaError_t launch_peer_gather(const PeerGather& g, int blocks, int threads, cudaStream_t s, bool pdl, bool lean) {
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.gridDim = dim3(blocks, 1, 1);
  cfg.blockDim = dim3(threads, 1, 1);
  cfg.dynamicSmemBytes = g.bulk ? 2 * kBulkChunk + 64 : 0;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (lean) {
    cfg.dynamicSmemBytes = 0;
    return cudaLaunchKernelEx(&cfg, peer_gather_kernel<true>, g);
  }
  return cudaLaunchKernelEx(&cfg, peer_gather_kernel<false>, g);
}

void* peer_gather_kernel_fn(bool lean) {
  return lean ? reinterpret_cast<void*>(peer_gather_kernel<true>) : reinterpret_cast<void*>(peer_gather_kernel<false>);
}

}  // namespace fc
