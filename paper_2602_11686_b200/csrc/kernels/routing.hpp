// Launchers of the routing / dispatch / combine kernels (routing.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels/fsep_types.cuh"

namespace fsep {

struct RouterArgs {
  const __nv_bfloat16* x;
  const __nv_bfloat16* wg;
  const float* bias;
  int T, H, E, K;
  int* topk_idx;
  float* topk_w;
  int* intra_rank;
  int* blk_hist;
};

struct DispatchArgs {
  const __nv_bfloat16* x;
  int T, H, K, E;
  const int* topk_idx;
  const int* intra_rank;
  const int* blk_base;
  const PlanTables* pt;
  PeerTable peers;
  uint32_t* slot_dst;
  int rank;  // source rank (row_src codes)
  const float* topk_w = nullptr;  // de-duplication: gate weights recorded per receive row
  int T_max = 0;
  bool dedupe = false;            // remote destinations get each token row once (PeerTable::stage)
};

void launch_router(const RouterArgs& a, cudaStream_t st);
void launch_block_scan(const int* blk_hist, int nblk, int E, int* blk_base, const PeerTable& peers, int rank,
                       int world, cudaStream_t st);
void launch_plan(const unsigned long long* R_all, const uint8_t* layout, int E, int N, int rank, PlanTables* pt,
                 long long row_capacity, bool local_first, unsigned* err, cudaStream_t st);
void launch_zero_pad(const PlanTables* pt, int C, int H, __nv_bfloat16* x_rows, __nv_bfloat16* dy_rows,
                     int* row_src, cudaStream_t st);
void launch_dispatch(const DispatchArgs& a, cudaStream_t st);
void launch_combine(int T, int H, int K, const float* topk_w, const __nv_bfloat16* tok_rows, __nv_bfloat16* out,
                    cudaStream_t st);
void launch_combine_bwd(int T, int H, int K, int E, const __nv_bfloat16* dout, const float* topk_w, const int* topk_idx,
                        const __nv_bfloat16* tok_rows, const uint32_t* slot_dst, const PeerTable& peers, float* dl,
                        __nv_bfloat16* dl_dense, int* rw_rows, int* rw_off, int rank, int T_max, bool dedupe,
                        cudaStream_t st);
// De-duplicated transfers: expand stage[src][t] into this rank's receive rows
// (row_w == nullptr: copy x rows; else dY rows = bf16(row_w[r] * stage row)).
void launch_expand_rows(const PlanTables* pt, long long capacity, const int* row_src, const __nv_bfloat16* stage,
                        const float* row_w, int rank, int H, int K, int T_max, __nv_bfloat16* rows, int num_sms,
                        cudaStream_t st);
bool use_tma_dispatch();
void launch_unpermute_bwd(int T, int H, int K, const int* topk_idx, const float* dl, const __nv_bfloat16* tok_rows,
                          const __nv_bfloat16* wg, __nv_bfloat16* dx, cudaStream_t st);
int router_wgrad_splits(int T);
void launch_router_wgrad(const __nv_bfloat16* x, int T, int H, int E, const __nv_bfloat16* dl_dense, int T_max,
                         const int* rw_rows, const int* rw_off, float* partial, float* dwg, int num_sms,
                         cudaStream_t st);
void launch_grad_reduce_scatter(const PlanTables* pt, const PeerTable& peers, int E, int rank, long long S,
                                long long flat, float* grad_shard, cudaStream_t st);
void launch_grad_rs_sum(const PlanTables* pt, const float* grad_full, const float* stage, int E, int N, int rank,
                        long long S, long long flat, float* grad_shard, cudaStream_t st);
void launch_pack_expert(const __nv_bfloat16* w1, const __nv_bfloat16* w3, const __nv_bfloat16* w2, int H, int F,
                        __nv_bfloat16* flat, cudaStream_t st);
void launch_unpack_grad(const float* chunk, long long lo, long long hi, int H, int F, float* dw1, float* dw3,
                        float* dw2, cudaStream_t st);

void launch_restore(const uint8_t* layout, int E, int N, int rank, int C, long long S, long long flat,
                    const PeerTable& peers, __nv_bfloat16* restored, int blocks_per_chunk, cudaStream_t st);

// SM push transport: all pieces of tasks[0, ntasks) (piece_bytes each, the last
// piece of a task shorter), grid-strided over `ctas` CTAs of 256 threads that use
// no shared memory and few registers -- they co-reside with the persistent GEMM
// (which polls the readiness flags), so the copies overlap it without deadlock.
// done: ntasks zero-initialised completion counters (zeroed here on `st`).
void launch_push_copies(const CopyTask* tasks, int ntasks, unsigned total_pieces, unsigned long long piece_bytes,
                        unsigned* done, int ctas, cudaStream_t st);

// Memory guards (256 B each, filled with `pattern`): *first_bad = min(index of an
// overwritten guard) -- initialise it to INT_MAX.
void launch_guard_check(const unsigned char* const* guards, int n, unsigned char pattern, int* first_bad,
                        cudaStream_t st);

// Cross-rank barrier for real multi-GPU mode (system-scope flags in peer memory).
// Bounded: after timeout_ns the kernel raises kErrBarrierTimeout in err (and flags[world]) and returns.
void launch_peer_barrier(unsigned int* const* peer_flags, int world, int rank, unsigned int epoch, unsigned* err,
                         unsigned long long timeout_ns, cudaStream_t st);

}  // namespace fsep
