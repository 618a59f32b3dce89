// Peer-memory data movement for the FSEP layer step over NVLink 5 / NVSwitch:
// the expert-granular shard restore (unshard) and the cross-rank barrier.
// Both read the layout and the peer pointer table on the device, so the whole
// step is enqueued without a host round-trip (and is CUDA-graph capturable).
#include <cuda_bf16.h>

#include "kernels/fsep_types.cuh"
#include "kernels/kernels.hpp"
#include "kernels/routing.hpp"

namespace fsep {

namespace {

// restored[c][p*S : (p+1)*S] = shard_p[e_c][0:S] for every peer p, where e_c is
// the c-th expert (ascending id) hosted by `rank` under the device layout.
// FSEP unshard at expert granularity: each device gathers
// only the C experts it will compute, chunk p from owner p.
__global__ void __launch_bounds__(256) restore_kernel(const uint8_t* __restrict__ layout, int E, int N, int rank,
                                                      long long S, long long flat, PeerTable peers,
                                                      __nv_bfloat16* __restrict__ restored) {
  __shared__ int s_expert;
  const int c = blockIdx.y, p = blockIdx.z;
  if (threadIdx.x == 0) {
    int seen = -1, found = -1;
    for (int e = 0; e < E && found < 0; ++e)
      if (layout[e * N + rank] && ++seen == c) found = e;
    s_expert = found;
  }
  __syncthreads();
  const int e = s_expert;
  if (e < 0) return;
  const uint4* __restrict__ src = reinterpret_cast<const uint4*>(peers.shard[p] + static_cast<long long>(e) * S);
  uint4* __restrict__ dst =
      reinterpret_cast<uint4*>(restored + static_cast<long long>(c) * flat + static_cast<long long>(p) * S);
  const long long n = S / 8;
  // 8 independent 16-B loads in flight per thread: peer (NVLink) loads are ~2 us away
  constexpr int U = 8;
  const long long stride = static_cast<long long>(gridDim.x) * 256;
  long long i = blockIdx.x * 256LL + threadIdx.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = src[i + u * stride];
#pragma unroll
    for (int u = 0; u < U; ++u) dst[i + u * stride] = v[u];
  }
  for (; i < n; i += stride) dst[i] = src[i];
}

// All-rank barrier: publish `epoch` into every peer's slot for this rank, then
// wait until every rank has published it here.  System-scope release/acquire
// orders the preceding peer stores of the step.  Bounded: after timeout_ns the
// kernel raises kErrBarrierTimeout (host-mapped, reported by the next
// mp_fsep_layer_* call as MP_ERR_DEVICE), records flags[world] and returns.
__global__ void peer_barrier_kernel(unsigned int* const* __restrict__ peer_flags, int world, int rank,
                                    unsigned int epoch, unsigned* err, unsigned long long timeout_ns) {
  const int p = threadIdx.x;
  if (p < world) {
    unsigned int* slot = peer_flags[p] + rank;
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(slot), "r"(epoch) : "memory");
    const unsigned int* mine = peer_flags[rank] + p;
    const unsigned long long t0 = globaltimer_ns();
    while (true) {
      unsigned int v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(mine) : "memory");
      if (static_cast<int>(v - epoch) >= 0) break;
      if (globaltimer_ns() - t0 > timeout_ns) {
        atomicOr(peer_flags[rank] + world, 1u);
        raise_err(err, kErrBarrierTimeout);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(256) push_copies_kernel(const CopyTask* __restrict__ tasks, int ntasks,
                                                         unsigned total_pieces, unsigned long long piece_bytes,
                                                         unsigned* __restrict__ done) {
  __shared__ int s_task;
  for (unsigned p = blockIdx.x; p < total_pieces; p += gridDim.x) {
    if (threadIdx.x == 0) {
      int t = 0;
      while (t + 1 < ntasks && tasks[t + 1].first_piece <= p) ++t;
      s_task = t;
    }
    __syncthreads();
    const CopyTask& tk = tasks[s_task];
    const unsigned long long off = static_cast<unsigned long long>(p - tk.first_piece) * piece_bytes;
    const unsigned long long len = min(piece_bytes, tk.bytes - off);
    const uint4* __restrict__ src = reinterpret_cast<const uint4*>(static_cast<const char*>(tk.src) + off);
    uint4* __restrict__ dst = reinterpret_cast<uint4*>(static_cast<char*>(tk.dst) + off);
    const long long n = static_cast<long long>(len / 16);
    // 4 independent 16-B loads (local HBM) in flight per thread, then 4 posted stores
    // (NVLink for a peer destination)
    constexpr int U = 4;
    long long i = threadIdx.x;
    for (; i + (U - 1) * 256 < n; i += U * 256) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = __ldg(src + i + u * 256);
#pragma unroll
      for (int u = 0; u < U; ++u) dst[i + u * 256] = v[u];
    }
    for (; i < n; i += 256) dst[i] = __ldg(src + i);
    __threadfence_system();  // this thread's stores are visible system-wide ...
    __syncthreads();         // ... for every thread of the CTA, before the completion count
    if (threadIdx.x == 0) {
      const unsigned pieces = static_cast<unsigned>((tk.bytes + piece_bytes - 1) / piece_bytes);
      unsigned prev;
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(done + s_task) : "memory");
      if (prev + 1 == pieces && tk.flag != nullptr)
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(tk.flag), "r"(tk.flag_val) : "memory");
    }
    __syncthreads();  // s_task is rewritten for the next piece
  }
}

// Memory guards: block g checks the 256-byte guard guards[g] (starts right after a
// buffer, so any byte alignment: byte loads) against the fill pattern and records the
// lowest failing guard index.
__global__ void guard_check_kernel(const unsigned char* const* __restrict__ guards, int n, unsigned char pattern,
                                   int* __restrict__ first_bad) {
  const int g = blockIdx.x;
  if (g >= n) return;
  bool ok = true;
  for (int i = static_cast<int>(threadIdx.x); i < 256; i += 32) ok &= guards[g][i] == pattern;
  if (!ok) atomicMin(first_bad, g);
}

}  // namespace

void launch_guard_check(const unsigned char* const* guards, int n, unsigned char pattern, int* first_bad,
                        cudaStream_t st) {
  if (n <= 0) return;
  guard_check_kernel<<<static_cast<unsigned>(n), 32, 0, st>>>(guards, n, pattern, first_bad);
  count_launch();
}

void launch_push_copies(const CopyTask* tasks, int ntasks, unsigned total_pieces, unsigned long long piece_bytes,
                        unsigned* done, int ctas, cudaStream_t st) {
  if (ntasks == 0 || total_pieces == 0) return;
  cudaMemsetAsync(done, 0, static_cast<size_t>(ntasks) * sizeof(unsigned), st);
  push_copies_kernel<<<static_cast<unsigned>(ctas), 256, 0, st>>>(tasks, ntasks, total_pieces, piece_bytes, done);
  count_launch();
}

void launch_restore(const uint8_t* layout, int E, int N, int rank, int C, long long S, long long flat,
                    const PeerTable& peers, __nv_bfloat16* restored, int blocks_per_chunk, cudaStream_t st) {
  restore_kernel<<<dim3(blocks_per_chunk, C, N), 256, 0, st>>>(layout, E, N, rank, S, flat, peers, restored);
  count_launch();
}

void launch_peer_barrier(unsigned int* const* peer_flags, int world, int rank, unsigned int epoch, unsigned* err,
                         unsigned long long timeout_ns, cudaStream_t st) {
  peer_barrier_kernel<<<1, 32, 0, st>>>(peer_flags, world, rank, epoch, err, timeout_ns);
  count_launch();
}

}  // namespace fsep
