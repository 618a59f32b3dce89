// Device-side data structures shared by the FSEP routing / dispatch / combine
// kernels and the host runtime.
//
// Receive layout on every device (expert-major, the grouped GEMM's A operand):
//   for each local slot c (hosted experts in ascending expert id):
//     rows [seg_off[c], seg_off[c] + seg_rows[c]) hold the tokens routed to that
//     expert, ordered by (source rank asc, token order within the source);
//     the segment is padded with zero rows up to a multiple of 128.
// A token-slot (t, k) of source rank i for expert e with rank r among
// (i, e)'s slots (ascending t) goes to the replica chosen by lite routing's
// share/remainder split (planner.cpp:277-282): host index h with
// cum[h] <= r < cum[h+1], row = row_base[h] + (r - cum[h]).
#pragma once
#include <cuda_bf16.h>

#include <cstdint>

namespace fsep {

constexpr int kMaxRanks = 16;
constexpr int kMaxExperts = 256;  // DeepSeek-V3-class layers (E = 256)
constexpr int kWaveSyncMax = 4096;  // wave-synchronisation counters per grouped-GEMM launch
constexpr int kBlockTokens = 64;  // router / ranking tile (8 warps x 8 tokens)
constexpr int kDLCols = 256;      // max width of the dense router-gradient matrix dL[t][e] (>= E)
// its width for E experts: 128 (one single-CTA M tile) up to 128 experts, else 256
__host__ __device__ constexpr int dl_cols(int E) { return E <= 128 ? 128 : 256; }
constexpr int kRouterWgradChunk = 1024;  // token rows per split-K group of the router wgrad GEMM

// Token-slot rows: every rank owns tok_rows[T_max * K][H] indexed by its own
// (token, k) slot.  The expert GEMMs' epilogues store their output rows (y in
// the forward, dX in the backward) straight into the owner's tok_rows over
// NVLink, guided by row_src, so combine / unpermute read only local HBM.
constexpr int kRowSrcShift = 26;  // row_src code = (source rank << 26) | (t * K + k); -1 = padding row
struct PeerTable {
  __nv_bfloat16* x_rows[kMaxRanks];
  __nv_bfloat16* dy_rows[kMaxRanks];
  __nv_bfloat16* tok_rows[kMaxRanks];  // [T_max*K][H] on each rank (y, later reused for dX)
  int* row_src[kMaxRanks];             // [row_capacity] origin of each receive row on each rank
  // Token de-duplication (K >= 4, N > 1): a token row crosses NVLink once per
  // destination device into stage[dst][src][t]; the destination expands it into
  // its slot rows (x rows in the forward, w_k-scaled dY rows in the backward).
  __nv_bfloat16* stage[kMaxRanks];     // [N][T_max][H] on each rank (null: no de-duplication)
  float* row_w[kMaxRanks];             // [row_capacity] gate weight w_k of each receive row
  unsigned long long* R_all[kMaxRanks];  // [N][E] on each rank
  float* grad_full[kMaxRanks];           // [C][3HF] restored-expert grads on each rank
  const __nv_bfloat16* shard[kMaxRanks]; // [E][S] FSEP shards on each rank
  uint64_t row_capacity;                 // rows of every receive buffer
};

// Device-detected step failures.  Each cause has its own word in host-mapped
// pinned memory (plain system-scope stores of 1: no host atomics needed over
// PCIe); the runtime reports a set word as MP_ERR_DEVICE at the next
// mp_fsep_layer_* call (mp_fsep_layer_check synchronises first).
enum ErrWord : int {
  kErrRecvOverflow = 0,     // a receive segment did not fit max_recv_rows (segments dropped)
  kErrBarrierTimeout = 1,   // a peer barrier timed out (a rank did not arrive)
  kErrRestoreTimeout = 2,   // a restored expert chunk's readiness flag never arrived
  kErrGuard = 3,            // host-detected: a buffer's memory guard was overwritten (mp_fsep_layer_check)
  kErrWords = 4,
};
__device__ __forceinline__ void raise_err(unsigned* err, int word) {
  if (err == nullptr) return;
  *reinterpret_cast<volatile unsigned*>(err + word) = 1u;
  __threadfence_system();
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// One copy of the SM push transport (comm.cu push_copies_kernel): `bytes` from
// src to dst (a peer's arena over NVLink, or local memory), split into pieces
// spread over the CTAs; once every piece has landed the CTA that finished last
// writes *flag = flag_val with a system-scope release (the destination's
// readiness word).  first_piece: prefix sum of the tasks' piece counts.
struct CopyTask {
  const void* src;
  void* dst;
  unsigned long long bytes;  // multiple of 16
  unsigned* flag;            // nullptr: no readiness flag
  unsigned flag_val;
  unsigned first_piece;
};

struct PlanTables {
  // global view (identical on all ranks)
  int n_hosts[kMaxExperts];
  int host_dev[kMaxExperts][kMaxRanks];  // ascending device ids
  int slot_of[kMaxExperts][kMaxRanks];   // local slot of expert e on device d (-1 if not hosted)
  // this rank as a source
  long long src_cum[kMaxExperts][kMaxRanks + 1];
  long long src_row_base[kMaxExperts][kMaxRanks];
  // this rank as a destination
  int slot_expert[kMaxExperts];
  int seg_rows[kMaxExperts];
  int seg_rows_pad[kMaxExperts];
  int seg_off[kMaxExperts];
  int total_rows;
  int status;  // bit 0: receive-buffer overflow
};

}  // namespace fsep
