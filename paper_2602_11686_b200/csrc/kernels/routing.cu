// Ranking, lite-routing assignment, dispatch/combine and their backward passes
// for the FSEP layer step (sm_100a, CUDA cores; all of these are HBM/NVLink-bound
// byte movers or tiny integer work).  The router itself is in router.cu.
//
// Bit-exactness contract with the CPU oracle (oracle/layer_oracle.py):
//  * token ranks within (source, expert) follow ascending token index, and the
//    replica split reproduces lite_routing (planner.cpp:277-282);
//  * every token-slot's destination (device, row) and the per-device segment
//    layout are integer functions of R, the layout and the ranks.
#include <algorithm>
#include <cstdlib>
#include <string>
#include <cuda_bf16.h>

#include <cfloat>
#include <stdexcept>

#include "kernels/fsep_types.cuh"
#include "kernels/sm100_ptx.cuh"
#include "kernels/kernels.hpp"
#include "kernels/routing.hpp"

namespace fsep {

namespace {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ void bf16x8_to_f32(const uint4& q, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

__device__ __forceinline__ uint4 f32_to_bf16x8(const float (&f)[8]) {
  uint4 q;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&q);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return q;
}

// Exclusive scan of per-block counts per expert -> block bases; R row of this
// rank is published into every rank's R_all (peer stores; local in N=1).
// Exclusive scan of the per-block expert counts (block b's base row for expert e
// among this rank's tokens) and the rank's histogram row R[rank][e], pushed to
// every rank's R_all.  One CTA per expert: chunked serial sums, a block-wide
// scan of the chunk totals, then the chunked writes.
__global__ void __launch_bounds__(256) block_scan_kernel(const int* __restrict__ blk_hist, int nblk, int E,
                                                         int* __restrict__ blk_base, PeerTable peers, int rank,
                                                         int world) {
  __shared__ int s_warp[8];
  const int e = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int per = (nblk + 255) / 256;
  const int b0 = min(nblk, tid * per), b1 = min(nblk, b0 + per);
  int sum = 0;
  for (int b = b0; b < b1; ++b) sum += blk_hist[static_cast<size_t>(b) * E + e];
  int inc = sum;  // inclusive warp scan
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += v;
  }
  if (lane == 31) s_warp[warp] = inc;
  __syncthreads();
  int before = 0;
  for (int w = 0; w < warp; ++w) before += s_warp[w];
  int base = before + inc - sum;  // exclusive prefix of this thread's chunk
  for (int b = b0; b < b1; ++b) {
    blk_base[static_cast<size_t>(b) * E + e] = base;
    base += blk_hist[static_cast<size_t>(b) * E + e];
  }
  if (tid == 255) {
    const long long total = static_cast<long long>(before) + inc;
    for (int p = 0; p < world; ++p) peers.R_all[p][static_cast<size_t>(rank) * E + e] = static_cast<unsigned long long>(total);
  }
}

__device__ __forceinline__ long long split_amount(long long tokens, int n, int t) {
  return tokens / n + (t < tokens % n ? 1 : 0);
}

// Lite routing on device (planner.cpp:238-287 for a single-node topology) and
// the receive layout of every device.  One block; E <= 128, N <= 16.
// Tokens source i sends to host index t of expert e: lite routing's even split
// (planner.cpp:277-282), or -- local-first variant -- everything to itself when
// i hosts a replica of e.
__device__ __forceinline__ long long route_amount(const unsigned long long* R_all, const uint8_t* layout,
                                                  const PlanTables* pt, int E, int N, int i, int e, int t, int nh,
                                                  bool local_first) {
  const long long tokens = static_cast<long long>(R_all[i * E + e]);
  if (local_first && layout[e * N + i]) return pt->host_dev[e][t] == i ? tokens : 0;
  return split_amount(tokens, nh, t);
}

__global__ void plan_kernel(const unsigned long long* __restrict__ R_all, const uint8_t* __restrict__ layout, int E,
                            int N, int rank, PlanTables* __restrict__ pt, long long row_capacity, bool local_first,
                            unsigned* err) {
  __shared__ int s_seg_off[kMaxRanks][kMaxExperts];
  const int tid = threadIdx.x;
  for (int e = tid; e < E; e += blockDim.x) {
    int n = 0;
    for (int d = 0; d < N; ++d)
      if (layout[e * N + d]) pt->host_dev[e][n++] = d;
    pt->n_hosts[e] = n;
  }
  __syncthreads();
  // per destination: slots in ascending expert order, padded segment offsets
  for (int d = tid; d < N; d += blockDim.x) {
    int c = 0;
    long long off = 0;
    for (int e = 0; e < E; ++e) {
      if (!layout[e * N + d]) {
        pt->slot_of[e][d] = -1;
        continue;
      }
      const int nh = pt->n_hosts[e];
      int t = 0;
      while (pt->host_dev[e][t] != d) ++t;
      long long rows = 0;
      for (int i = 0; i < N; ++i) rows += route_amount(R_all, layout, pt, E, N, i, e, t, nh, local_first);
      pt->slot_of[e][d] = c;
      s_seg_off[d][c] = static_cast<int>(off);
      if (d == rank) {
        pt->slot_expert[c] = e;
        pt->seg_off[c] = static_cast<int>(off);
        // A segment that does not fit the receive buffer is dropped (the GEMMs see 0
        // rows; dispatch skips rows past the capacity) and status flags the step.
        const bool fits = off + (rows + 127) / 128 * 128 <= row_capacity;
        pt->seg_rows[c] = fits ? static_cast<int>(rows) : 0;
        pt->seg_rows_pad[c] = fits ? static_cast<int>((rows + 127) / 128 * 128) : 0;
      }
      off += (rows + 127) / 128 * 128;
      ++c;
    }
    if (d == rank) {
      pt->total_rows = static_cast<int>(off);
      pt->status = off > row_capacity ? 1 : 0;
      if (off > row_capacity) raise_err(err, kErrRecvOverflow);
    }
  }
  __syncthreads();
  // this rank as a source: per expert, cumulative split and destination rows
  for (int e = tid; e < E; e += blockDim.x) {
    const int nh = pt->n_hosts[e];
    long long cum = 0;
    for (int t = 0; t < nh; ++t) {
      const int d = pt->host_dev[e][t];
      long long before = 0;  // rows from lower-ranked sources on d for e
      for (int i = 0; i < rank; ++i) before += route_amount(R_all, layout, pt, E, N, i, e, t, nh, local_first);
      pt->src_cum[e][t] = cum;
      pt->src_row_base[e][t] = s_seg_off[d][pt->slot_of[e][d]] + before;
      cum += route_amount(R_all, layout, pt, E, N, rank, e, t, nh, local_first);
    }
    pt->src_cum[e][nh] = cum;
  }
}

// Zero the padding rows of this rank's receive buffers (X rows and dY rows) so
// the GEMMs may run over padded segments and the wgrad reduction stays exact.
__global__ void zero_pad_kernel(const PlanTables* __restrict__ pt, int C, int H, __nv_bfloat16* x_rows,
                                __nv_bfloat16* dy_rows, int* row_src) {
  const int c = blockIdx.y;
  if (c >= C) return;
  const int rows = pt->seg_rows[c], pad = pt->seg_rows_pad[c] - rows;
  if (blockIdx.x == 0 && static_cast<int>(threadIdx.x) < pad) row_src[pt->seg_off[c] + rows + threadIdx.x] = -1;
  const size_t base = static_cast<size_t>(pt->seg_off[c] + rows) * H;
  const size_t n = static_cast<size_t>(pad) * H / 8;
  uint4 z = make_uint4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    reinterpret_cast<uint4*>(x_rows + base)[i] = z;
    reinterpret_cast<uint4*>(dy_rows + base)[i] = z;
  }
}

// ------------------------------------------------------------------ dispatch
// Warp per token: resolve each slot's (device, row), record it, copy the token
// row once from HBM and store it K times (local HBM or a peer over NVLink).
template <int CH>
__global__ void __launch_bounds__(256) dispatch_kernel(const __nv_bfloat16* __restrict__ x, int T, int K, int E,
                                                       const int* __restrict__ topk_idx,
                                                       const int* __restrict__ intra_rank,
                                                       const int* __restrict__ blk_base,
                                                       const PlanTables* __restrict__ pt, PeerTable peers,
                                                       uint32_t* __restrict__ slot_dst, int src_rank) {
  constexpr int H = CH * 256;
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  uint4* dst_row[8];
  for (int k = 0; k < K; ++k) {
    const int e = topk_idx[static_cast<size_t>(t) * K + k];
    const long long r = blk_base[static_cast<size_t>(t / kBlockTokens) * E + e] + intra_rank[static_cast<size_t>(t) * K + k];
    int h = 0;
    while (pt->src_cum[e][h + 1] <= r) ++h;
    const int d = pt->host_dev[e][h];
    const long long row = pt->src_row_base[e][h] + (r - pt->src_cum[e][h]);
    const bool fits = static_cast<uint64_t>(row) < peers.row_capacity;
    if (lane == 0) {
      slot_dst[static_cast<size_t>(t) * K + k] = (static_cast<uint32_t>(d) << 24) | static_cast<uint32_t>(row);
      if (fits) peers.row_src[d][row] = (src_rank << kRowSrcShift) | (t * K + k);
    }
    dst_row[k] = fits ? reinterpret_cast<uint4*>(peers.x_rows[d] + static_cast<size_t>(row) * H) : nullptr;
  }
  const uint4* src = reinterpret_cast<const uint4*>(x + static_cast<size_t>(t) * H);
  uint4 v[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) v[c] = __ldg(src + c * 32 + lane);
  for (int k = 0; k < K; ++k) {
    if (!dst_row[k]) continue;
#pragma unroll
    for (int c = 0; c < CH; ++c) dst_row[k][c * 32 + lane] = v[c];
  }
}

// TMA-engine dispatch: per warp a ring of kDispatchBufs row buffers in shared
// memory; lane 0 bulk-loads token rows (local HBM) ahead and bulk-stores each
// row to its K destination rows (local HBM or peers over NVLink), so the
// copies run on the TMA engine with many rows in flight per SM instead of
// through per-thread 16-B stores.
constexpr int kDispatchWarps = 4;
template <int CH>
constexpr int dispatch_bufs() { return CH >= 16 ? 3 : (CH >= 8 ? 6 : 8); }
template <int CH>
constexpr size_t dispatch_smem() {
  return static_cast<size_t>(kDispatchWarps) * dispatch_bufs<CH>() * (CH * 512 + 16);
}

template <int CH>
__global__ void __launch_bounds__(kDispatchWarps * 32) dispatch_tma_kernel(
    const __nv_bfloat16* __restrict__ x, int T, int K, int E, const int* __restrict__ topk_idx,
    const int* __restrict__ intra_rank, const int* __restrict__ blk_base, const PlanTables* __restrict__ pt,
    PeerTable peers, uint32_t* __restrict__ slot_dst, int src_rank, const float* __restrict__ topk_w, int T_max,
    bool dedupe) {
  using namespace ptx;
  constexpr int H = CH * 256;
  constexpr uint32_t RB = H * 2;
  constexpr int NB = dispatch_bufs<CH>();
  extern __shared__ __align__(128) uint8_t dsm[];
  const int warp = static_cast<int>(threadIdx.x >> 5), lane = static_cast<int>(threadIdx.x & 31);
  uint8_t* buf = dsm + static_cast<size_t>(warp) * NB * RB;
  uint64_t* bar = reinterpret_cast<uint64_t*>(dsm + static_cast<size_t>(kDispatchWarps) * NB * RB) + warp * NB;
  const int gw = blockIdx.x * kDispatchWarps + warp, nw = gridDim.x * kDispatchWarps;
  if (lane == 0) {
    for (int b = 0; b < NB; ++b) mbar_init(&bar[b], 1);
    fence_mbar_init();
  }
  __syncwarp();
  auto issue = [&](int j) {  // bulk-load token gw + j*nw into buffer j % NB
    const int t = gw + j * nw;
    if (t >= T) return;
    uint64_t* b = &bar[j % NB];
    mbar_arrive_expect_tx(b, RB);
    bulk_g2s(buf + static_cast<size_t>(j % NB) * RB, x + static_cast<size_t>(t) * H, RB, b);
  };
  if (lane == 0)
    for (int j = 0; j < NB; ++j) issue(j);
  for (int j = 0;; ++j) {
    const int t = gw + j * nw;
    if (t >= T) break;
    // lane k resolves slot k's destination (same rule as dispatch_kernel)
    unsigned long long dst = 0;
    int rdev = -1;  // de-duplicated remote destination device of slot k
    if (lane < K) {
      const int k = lane;
      const int e = topk_idx[static_cast<size_t>(t) * K + k];
      const long long r = blk_base[static_cast<size_t>(t / kBlockTokens) * E + e] + intra_rank[static_cast<size_t>(t) * K + k];
      int h = 0;
      while (pt->src_cum[e][h + 1] <= r) ++h;
      const int d = pt->host_dev[e][h];
      const long long row = pt->src_row_base[e][h] + (r - pt->src_cum[e][h]);
      slot_dst[static_cast<size_t>(t) * K + k] = (static_cast<uint32_t>(d) << 24) | static_cast<uint32_t>(row);
      if (static_cast<uint64_t>(row) < peers.row_capacity) {
        peers.row_src[d][row] = (src_rank << kRowSrcShift) | (t * K + k);
        if (dedupe) {
          peers.row_w[d][row] = topk_w[static_cast<size_t>(t) * K + k];
          if (d != src_rank) rdev = d;
        }
        if (rdev < 0) dst = reinterpret_cast<unsigned long long>(peers.x_rows[d] + static_cast<size_t>(row) * H);
      }
    }
    unsigned long long dk[8];
    int rk[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      dk[k] = __shfl_sync(0xffffffffu, dst, k);
      rk[k] = __shfl_sync(0xffffffffu, rdev, k);
    }
    if (lane == 0) {
      mbar_wait(&bar[j % NB], (j / NB) & 1);
      const uint8_t* src = buf + static_cast<size_t>(j % NB) * RB;
      for (int k = 0; k < K; ++k) {
        if (dk[k]) bulk_s2g(reinterpret_cast<void*>(dk[k]), src, RB);
        if (rk[k] >= 0) {  // once per remote device: the token row into its staging area
          bool seen = false;
          for (int q = 0; q < k; ++q) seen |= rk[q] == rk[k];
          if (!seen)
            bulk_s2g(peers.stage[rk[k]] + (static_cast<size_t>(src_rank) * T_max + t) * H, src, RB);
        }
      }
      bulk_commit();
      if (j >= 1) {  // buffer of token j-1 is free once its stores have read it
        bulk_wait_read<1>();
        issue(j - 1 + NB);
      }
    }
    __syncwarp();
  }
  if (lane == 0) bulk_wait<0>();
}

__device__ __forceinline__ const uint4* row_ptr(__nv_bfloat16* const* bufs, uint32_t code, int H) {
  return reinterpret_cast<const uint4*>(bufs[code >> 24] + static_cast<size_t>(code & 0xFFFFFFu) * H);
}

// ------------------------------------------------------------------ combine
// out[t] = sum_k w[t,k] * y[slot(t,k)]  (fp32 accumulate in k order, bf16 out)
template <int CH>
__global__ void __launch_bounds__(256) combine_kernel(int T, int K, const float* __restrict__ topk_w,
                                                      const __nv_bfloat16* __restrict__ tok_rows,
                                                      __nv_bfloat16* __restrict__ out) {
  constexpr int H = CH * 256;
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  uint4* o = reinterpret_cast<uint4*>(out + static_cast<size_t>(t) * H);
#pragma unroll
  for (int c0 = 0; c0 < CH; c0 += 4) {
    float acc[4][8];
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[c][j] = 0.f;
    for (int k = 0; k < K; ++k) {
      const float w = topk_w[static_cast<size_t>(t) * K + k];
      const uint4* y = reinterpret_cast<const uint4*>(tok_rows + (static_cast<size_t>(t) * K + k) * H);
      uint4 q[4];
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (c0 + c < CH) q[c] = y[(c0 + c) * 32 + lane];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (c0 + c >= CH) break;
        float f[8];
        bf16x8_to_f32(q[c], f);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[c][j] = __fmaf_rn(w, f[j], acc[c][j]);
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (c0 + c < CH) o[(c0 + c) * 32 + lane] = f32_to_bf16x8(acc[c]);
  }
}

// ------------------------------------------------------------- combine bwd
// dy[slot(t,k)] = w[t,k] * dout[t]   (scattered back to the expert's device)
// dw[t,k]       = <dout[t], y[slot(t,k)]>
// dl[t,k]       = w_k (dw_k - sum_j w_j dw_j)       (softmax-over-top-k backward)
// Also scatters dl into the dense bf16 matrix dL[t][e] (kDLCols wide, pre-zeroed)
// that feeds the router weight-gradient GEMM, and (block 0) writes that GEMM's
// split-K group table: groups of kRouterWgradChunk token rows.
template <int CH>
__global__ void __launch_bounds__(256) combine_bwd_kernel(int T, int K, const __nv_bfloat16* __restrict__ dout,
                                                          const float* __restrict__ topk_w,
                                                          const int* __restrict__ topk_idx,
                                                          const __nv_bfloat16* __restrict__ tok_rows,
                                                          const uint32_t* __restrict__ slot_dst, PeerTable peers,
                                                          float* __restrict__ dl, __nv_bfloat16* __restrict__ dl_dense,
                                                          int* __restrict__ rw_rows, int* __restrict__ rw_off, int dlc,
                                                          int src_rank, int T_max, bool dedupe) {
  constexpr int H = CH * 256;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const int tpad = (T + 127) / 128 * 128;
    for (int g = 0, r = 0; r < tpad; ++g, r += kRouterWgradChunk) {
      rw_off[g] = r;
      rw_rows[g] = min(kRouterWgradChunk, tpad - r);
    }
  }
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  const uint4* g = reinterpret_cast<const uint4*>(dout + static_cast<size_t>(t) * H);
  float dot[8];
  float w[8];
  // per slot: write the scaled dY row directly (local, or every slot without
  // de-duplication), or -- de-duplicated remote device, first slot on it -- send
  // the raw dout row once into that device's staging area (expanded there)
  bool direct[8], first[8];
  int dev[8];
  for (int k = 0; k < K; ++k) {
    dot[k] = 0.f;
    w[k] = topk_w[static_cast<size_t>(t) * K + k];
    const uint32_t code = slot_dst[static_cast<size_t>(t) * K + k];
    dev[k] = static_cast<int>(code >> 24);
    const bool valid = (code & 0xFFFFFFu) < peers.row_capacity;  // dropped slots (receive overflow) are skipped
    const bool remote = dedupe && dev[k] != src_rank;
    direct[k] = valid && !remote;
    bool seen = false;
    for (int q = 0; q < k; ++q) seen |= first[q] && dev[q] == dev[k];
    first[k] = valid && remote && !seen;
  }
#pragma unroll
  for (int c0 = 0; c0 < CH; c0 += 4) {
    float gf[4][8];
    uint4 graw[4];
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (c0 + c < CH) {
        graw[c] = __ldg(g + (c0 + c) * 32 + lane);
        bf16x8_to_f32(graw[c], gf[c]);
      }
    for (int k = 0; k < K; ++k) {
      const uint32_t code = slot_dst[static_cast<size_t>(t) * K + k];
      const uint4* y = reinterpret_cast<const uint4*>(tok_rows + (static_cast<size_t>(t) * K + k) * H);
      uint4* dy = const_cast<uint4*>(row_ptr(peers.dy_rows, code, H));
      uint4 q[4];
#pragma unroll
      for (int c = 0; c < 4; ++c)
        if (c0 + c < CH) q[c] = y[(c0 + c) * 32 + lane];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (c0 + c >= CH) break;
        float f[8], s[8];
        bf16x8_to_f32(q[c], f);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          dot[k] = __fmaf_rn(gf[c][j], f[j], dot[k]);
          s[j] = w[k] * gf[c][j];
        }
        if (direct[k]) dy[(c0 + c) * 32 + lane] = f32_to_bf16x8(s);
      }
      if (first[k]) {
        uint4* st = reinterpret_cast<uint4*>(peers.stage[dev[k]] + (static_cast<size_t>(src_rank) * T_max + t) * H);
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (c0 + c < CH) st[(c0 + c) * 32 + lane] = graw[c];
      }
    }
  }
  float dw[8];
  float mix = 0.f;
  for (int k = 0; k < K; ++k) {
    dw[k] = warp_sum(dot[k]);
    mix += w[k] * dw[k];
  }
  if (lane == 0)
    for (int k = 0; k < K; ++k) {
      const float v = w[k] * (dw[k] - mix);
      dl[static_cast<size_t>(t) * K + k] = v;
      dl_dense[static_cast<size_t>(t) * dlc + topk_idx[static_cast<size_t>(t) * K + k]] = __float2bfloat16_rn(v);
    }
}

// ------------------------------------------------------------- expansion
// De-duplicated transfers land once per (source, token) in stage[src][t]; every
// receive row whose source is another rank copies its token row from there
// (forward: x rows), or -- with row weights -- writes bf16(w_k * dout) (backward:
// dY rows, the same fp32 product combine_bwd forms for local slots).
template <int CH>
__global__ void __launch_bounds__(256) expand_rows_kernel(const PlanTables* __restrict__ pt, long long capacity,
                                                          const int* __restrict__ row_src,
                                                          const __nv_bfloat16* __restrict__ stage,
                                                          const float* __restrict__ row_w, int rank, int K,
                                                          int T_max, __nv_bfloat16* __restrict__ rows) {
  constexpr int H = CH * 256;
  const int lane = threadIdx.x & 31;
  const long long n = min(static_cast<long long>(pt->total_rows), capacity);
  for (long long r = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < n;
       r += (static_cast<long long>(gridDim.x) * blockDim.x) >> 5) {
    const int code = row_src[r];
    if (code < 0) continue;
    const int s = code >> kRowSrcShift;
    if (s == rank) continue;  // written directly by the local dispatch / combine-bwd
    const int t = (code & ((1 << kRowSrcShift) - 1)) / K;
    const uint4* src = reinterpret_cast<const uint4*>(stage + (static_cast<size_t>(s) * T_max + t) * H);
    uint4* dst = reinterpret_cast<uint4*>(rows + static_cast<size_t>(r) * H);
    if (row_w == nullptr) {
#pragma unroll
      for (int c = 0; c < CH; ++c) dst[c * 32 + lane] = src[c * 32 + lane];
    } else {
      const float w = row_w[r];
#pragma unroll
      for (int c = 0; c < CH; ++c) {
        float f[8], o[8];
        bf16x8_to_f32(src[c * 32 + lane], f);
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = w * f[j];
        dst[c * 32 + lane] = f32_to_bf16x8(o);
      }
    }
  }
}

// ----------------------------------------------------------- unpermute bwd
// dx[t] = sum_k dX_rows[slot(t,k)] + sum_k dl[t,k] * wg[e_k]   (router path)
template <int CH>
__global__ void __launch_bounds__(256) unpermute_bwd_kernel(int T, int K, const int* __restrict__ topk_idx,
                                                            const float* __restrict__ dl,
                                                            const __nv_bfloat16* __restrict__ tok_rows,
                                                            const __nv_bfloat16* __restrict__ wg,
                                                            __nv_bfloat16* __restrict__ dx) {
  constexpr int H = CH * 256;
  const int t = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  uint4* o = reinterpret_cast<uint4*>(dx + static_cast<size_t>(t) * H);
#pragma unroll
  for (int c0 = 0; c0 < CH; c0 += 4) {
    float acc[4][8];
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[c][j] = 0.f;
    for (int k = 0; k < K; ++k) {
      const uint4* r = reinterpret_cast<const uint4*>(tok_rows + (static_cast<size_t>(t) * K + k) * H);
      const float d = dl[static_cast<size_t>(t) * K + k];
      const uint4* w = reinterpret_cast<const uint4*>(wg + static_cast<size_t>(topk_idx[static_cast<size_t>(t) * K + k]) * H);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (c0 + c >= CH) break;
        float f[8], wf[8];
        bf16x8_to_f32(r[(c0 + c) * 32 + lane], f);
        bf16x8_to_f32(__ldg(w + (c0 + c) * 32 + lane), wf);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[c][j] += f[j] + d * wf[j];
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c)
      if (c0 + c < CH) o[(c0 + c) * 32 + lane] = f32_to_bf16x8(acc[c]);
  }
}

// ------------------------------------------------------------ router wgrad
// dWg = dL^T x runs as a split-K tcgen05 GEMM (K-grouped over token chunks, one
// [kDLCols x H] fp32 partial per chunk); the partials' first E rows are summed
// here in fixed chunk order (deterministic).
__global__ void router_wgrad_reduce_kernel(const float* __restrict__ partial, int splits, int EH, int H, int dlc,
                                           float* __restrict__ dwg) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= EH) return;
  float s = 0.f;
  for (int p = 0; p < splits; ++p) s += partial[static_cast<size_t>(p) * dlc * H + i];
  dwg[i] = s;
}

// ------------------------------------------------------------ grad RS
// Owner `rank` sums chunk `rank` of every expert's gradient over the devices
// that hosted a replica this step (ascending device order -> deterministic),
// reading the replicas' fp32 gradients in place (peer loads over NVLink).
__global__ void grad_reduce_scatter_kernel(const PlanTables* __restrict__ pt, PeerTable peers, int E, int rank,
                                           long long S, long long flat, float* __restrict__ grad_shard) {
  const int e = blockIdx.y;
  const int nh = pt->n_hosts[e];
  const float4* src[kMaxRanks];
  for (int h = 0; h < nh; ++h) {
    const int d = pt->host_dev[e][h];
    src[h] = reinterpret_cast<const float4*>(peers.grad_full[d] + static_cast<long long>(pt->slot_of[e][d]) * flat +
                                             static_cast<long long>(rank) * S);
  }
  float4* dst = reinterpret_cast<float4*>(grad_shard + static_cast<long long>(e) * S);
  // 4 elements per thread per round, all replicas' loads issued before the sums
  // (peer loads are ~2 us away); summation order stays ascending-device.
  constexpr int U = 4;
  const long long n = S / 4;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += U * stride) {
    float4 a[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i0 + u * stride < n) a[u] = src[0][i0 + u * stride];
    for (int h = 1; h < nh; ++h) {
      float4 b[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i0 + u * stride < n) b[u] = src[h][i0 + u * stride];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        a[u].x += b[u].x;
        a[u].y += b[u].y;
        a[u].z += b[u].z;
        a[u].w += b[u].w;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i0 + u * stride < n) dst[i0 + u * stride] = a[u];
  }
}

// Owner-side sum of the grad reduce-scatter when the replicas' chunks were
// gathered by copy engines into stage[e][h] (h = hosting device): ascending-device
// order, the local replica read in place.  Deterministic, HBM-bound.
__global__ void grad_rs_sum_kernel(const PlanTables* __restrict__ pt, const float* __restrict__ grad_full,
                                   const float* __restrict__ stage, int N, int rank, long long S, long long flat,
                                   float* __restrict__ grad_shard) {
  const int e = blockIdx.y;
  const int nh = pt->n_hosts[e];
  const float4* src[kMaxRanks];
  for (int h = 0; h < nh; ++h) {
    const int d = pt->host_dev[e][h];
    src[h] = d == rank ? reinterpret_cast<const float4*>(grad_full + static_cast<long long>(pt->slot_of[e][d]) * flat +
                                                         static_cast<long long>(rank) * S)
                       : reinterpret_cast<const float4*>(stage + (static_cast<long long>(e) * N + d) * S);
  }
  float4* dst = reinterpret_cast<float4*>(grad_shard + static_cast<long long>(e) * S);
  const long long n = S / 4;
  // 4 float4 per thread per source in flight (streaming loads / stores: nothing
  // here is re-read), summed in ascending host order
  constexpr int U = 4;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    float4 a[U];
#pragma unroll
    for (int u = 0; u < U; ++u) a[u] = __ldcs(src[0] + i + u * stride);
    for (int h = 1; h < nh; ++h) {
      float4 b[U];
#pragma unroll
      for (int u = 0; u < U; ++u) b[u] = __ldcs(src[h] + i + u * stride);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        a[u].x += b[u].x;
        a[u].y += b[u].y;
        a[u].z += b[u].z;
        a[u].w += b[u].w;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) __stcs(dst + i + u * stride, a[u]);
  }
  for (; i < n; i += stride) {
    float4 a = __ldcs(src[0] + i);
    for (int h = 1; h < nh; ++h) {
      const float4 b = __ldcs(src[h] + i);
      a.x += b.x;
      a.y += b.y;
      a.z += b.z;
      a.w += b.w;
    }
    __stcs(dst + i, a);
  }
}

// ------------------------------------------------------------ weight packing
// flat[3HF] = [W13 interleaved: rows 256b+q (q<128) = w1[128b+q], 256b+128+q = w3[128b+q]; W2]
__global__ void pack_expert_kernel(const __nv_bfloat16* __restrict__ w1, const __nv_bfloat16* __restrict__ w3,
                                   const __nv_bfloat16* __restrict__ w2, int H, int F,
                                   __nv_bfloat16* __restrict__ flat) {
  const long long n13 = 2LL * F * H, total = 3LL * F * H;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < total; i += static_cast<long long>(gridDim.x) * 256) {
    if (i < n13) {
      const long long row = i / H, col = i % H;
      const long long b = row / 256, q = row % 256;
      const long long src_row = b * 128 + (q % 128);
      flat[i] = (q < 128 ? w1 : w3)[src_row * H + col];
    } else {
      flat[i] = w2[i - n13];
    }
  }
}

// Inverse of pack_expert for fp32 gradients, restricted to [lo, hi) of the flat
// vector (a rank's shard chunk); elements outside are not written.
__global__ void unpack_grad_kernel(const float* __restrict__ chunk, long long lo, long long hi, int H, int F,
                                   float* __restrict__ dw1, float* __restrict__ dw3, float* __restrict__ dw2) {
  const long long n13 = 2LL * F * H;
  for (long long i = lo + blockIdx.x * 256LL + threadIdx.x; i < hi; i += static_cast<long long>(gridDim.x) * 256) {
    const float v = chunk[i - lo];
    if (i < n13) {
      const long long row = i / H, col = i % H;
      const long long b = row / 256, q = row % 256;
      const long long dst_row = b * 128 + (q % 128);
      (q < 128 ? dw1 : dw3)[dst_row * H + col] = v;
    } else {
      dw2[i - n13] = v;
    }
  }
}

}  // namespace

// ------------------------------------------------------------------ launchers
#define FSEP_CH_SWITCH(CHV, ...)                                                         \
  switch (CHV) {                                                                         \
    case 1: { constexpr int CH = 1; __VA_ARGS__; } break;                                \
    case 2: { constexpr int CH = 2; __VA_ARGS__; } break;                                \
    case 3: { constexpr int CH = 3; __VA_ARGS__; } break;                                \
    case 4: { constexpr int CH = 4; __VA_ARGS__; } break;                                \
    case 5: { constexpr int CH = 5; __VA_ARGS__; } break;                                \
    case 6: { constexpr int CH = 6; __VA_ARGS__; } break;                                \
    case 8: { constexpr int CH = 8; __VA_ARGS__; } break;                                \
    case 10: { constexpr int CH = 10; __VA_ARGS__; } break;                              \
    case 12: { constexpr int CH = 12; __VA_ARGS__; } break;                              \
    case 14: { constexpr int CH = 14; __VA_ARGS__; } break;                              \
    case 16: { constexpr int CH = 16; __VA_ARGS__; } break;                              \
    case 20: { constexpr int CH = 20; __VA_ARGS__; } break;                              \
    case 24: { constexpr int CH = 24; __VA_ARGS__; } break;                              \
    case 28: { constexpr int CH = 28; __VA_ARGS__; } break;                              \
    case 32: { constexpr int CH = 32; __VA_ARGS__; } break;                              \
    default: throw std::runtime_error("hidden size must be 256 * {1-6,8,10,12,14,16,20,24,28,32}"); \
  }

void launch_block_scan(const int* blk_hist, int nblk, int E, int* blk_base, const PeerTable& peers, int rank,
                       int world, cudaStream_t st) {
  block_scan_kernel<<<E, 256, 0, st>>>(blk_hist, nblk, E, blk_base, peers, rank, world);
  count_launch();
}

void launch_plan(const unsigned long long* R_all, const uint8_t* layout, int E, int N, int rank, PlanTables* pt,
                 long long row_capacity, bool local_first, unsigned* err, cudaStream_t st) {
  plan_kernel<<<1, 128, 0, st>>>(R_all, layout, E, N, rank, pt, row_capacity, local_first, err);
  count_launch();
}

void launch_zero_pad(const PlanTables* pt, int C, int H, __nv_bfloat16* x_rows, __nv_bfloat16* dy_rows, int* row_src,
                     cudaStream_t st) {
  zero_pad_kernel<<<dim3(16, C), 256, 0, st>>>(pt, C, H, x_rows, dy_rows, row_src);
  count_launch();
}

bool use_tma_dispatch() {
  static const bool on = [] {
    const char* v = std::getenv("FSEP_DISPATCH");
    return !(v && std::string(v) == "simt");
  }();
  return on;
}

void launch_dispatch(const DispatchArgs& a, cudaStream_t st) {
  if (a.T == 0) return;
  if (use_tma_dispatch()) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    FSEP_CH_SWITCH(a.H / 256, {
      constexpr size_t smem = dispatch_smem<CH>() + kDispatchWarps * dispatch_bufs<CH>() * 8;
      set_smem_attr(reinterpret_cast<const void*>(dispatch_tma_kernel<CH>), static_cast<int>(smem));
      static const int per_sm = [] {  // FSEP_DISPATCH_CTAS_PER_SM: resident dispatch CTAs per SM (A/B)
        const char* v = std::getenv("FSEP_DISPATCH_CTAS_PER_SM");
        return v ? std::max(1, std::atoi(v)) : 1;
      }();
      const int blocks = std::min(sms * per_sm, (a.T + kDispatchWarps - 1) / kDispatchWarps);
      dispatch_tma_kernel<CH><<<blocks, kDispatchWarps * 32, smem, st>>>(
          a.x, a.T, a.K, a.E, a.topk_idx, a.intra_rank, a.blk_base, a.pt, a.peers, a.slot_dst, a.rank, a.topk_w,
          a.T_max, a.dedupe);
    });
  } else {
    FSEP_CH_SWITCH(a.H / 256, dispatch_kernel<CH><<<(a.T + 7) / 8, 256, 0, st>>>(
                                  a.x, a.T, a.K, a.E, a.topk_idx, a.intra_rank, a.blk_base, a.pt, a.peers, a.slot_dst,
                                  a.rank));
  }
  count_launch();
}

void launch_combine(int T, int H, int K, const float* topk_w, const __nv_bfloat16* tok_rows, __nv_bfloat16* out,
                    cudaStream_t st) {
  if (T == 0) return;
  FSEP_CH_SWITCH(H / 256, combine_kernel<CH><<<(T + 7) / 8, 256, 0, st>>>(T, K, topk_w, tok_rows, out));
  count_launch();
}

void launch_combine_bwd(int T, int H, int K, int E, const __nv_bfloat16* dout, const float* topk_w, const int* topk_idx,
                        const __nv_bfloat16* tok_rows, const uint32_t* slot_dst, const PeerTable& peers, float* dl,
                        __nv_bfloat16* dl_dense, int* rw_rows, int* rw_off, int rank, int T_max, bool dedupe,
                        cudaStream_t st) {
  if (T == 0) return;
  const size_t tpad = (static_cast<size_t>(T) + 127) / 128 * 128;
  const int dlc = dl_cols(E);
  cudaMemsetAsync(dl_dense, 0, tpad * dlc * sizeof(__nv_bfloat16), st);
  FSEP_CH_SWITCH(H / 256, combine_bwd_kernel<CH><<<(T + 7) / 8, 256, 0, st>>>(
                              T, K, dout, topk_w, topk_idx, tok_rows, slot_dst, peers, dl, dl_dense, rw_rows, rw_off,
                              dlc, rank, T_max, dedupe));
  count_launch();
}

void launch_unpermute_bwd(int T, int H, int K, const int* topk_idx, const float* dl, const __nv_bfloat16* tok_rows,
                          const __nv_bfloat16* wg, __nv_bfloat16* dx, cudaStream_t st) {
  if (T == 0) return;
  FSEP_CH_SWITCH(H / 256, unpermute_bwd_kernel<CH><<<(T + 7) / 8, 256, 0, st>>>(T, K, topk_idx, dl, tok_rows, wg, dx));
  count_launch();
}

void launch_expand_rows(const PlanTables* pt, long long capacity, const int* row_src, const __nv_bfloat16* stage,
                        const float* row_w, int rank, int H, int K, int T_max, __nv_bfloat16* rows, int num_sms,
                        cudaStream_t st) {
  FSEP_CH_SWITCH(H / 256, expand_rows_kernel<CH><<<num_sms * 8, 256, 0, st>>>(pt, capacity, row_src, stage, row_w,
                                                                             rank, K, T_max, rows));
  count_launch();
}

int router_wgrad_splits(int T) {
  const int tpad = (T + 127) / 128 * 128;
  return tpad == 0 ? 1 : (tpad + kRouterWgradChunk - 1) / kRouterWgradChunk;
}

void launch_router_wgrad(const __nv_bfloat16* x, int T, int H, int E, const __nv_bfloat16* dl_dense, int T_max,
                         const int* rw_rows, const int* rw_off, float* partial, float* dwg, int num_sms,
                         cudaStream_t st) {
  const int splits = router_wgrad_splits(T);
  const int dlc = dl_cols(E);
  if (T > 0) {
    // dL [rows][kDLCols] and x [rows][H] are both MN-major operands of the K-grouped GEMM
    const uint64_t tmax_pad = (static_cast<uint64_t>(T_max) + 127) / 128 * 128;
    const CUtensorMap ta = make_tmap_2d(dl_dense, dlc, tmax_pad, dlc, 64, 64);
    const CUtensorMap tb = make_tmap_2d(x, H, static_cast<uint64_t>(T), H, 64, 64);
    GroupedGemmArgs g{};
    g.num_groups = splits;
    g.group_rows = rw_rows;
    g.group_off = rw_off;
    g.M = dlc;
    g.N = H;
    g.out = partial;
    g.ldo = H;
    g.out_group_stride = static_cast<long long>(dlc) * H;
    launch_grouped_gemm(GemmKind::kBwdWgrad, ta, tb, g, num_sms, st);
  } else {
    cudaMemsetAsync(partial, 0, static_cast<size_t>(dlc) * H * sizeof(float), st);
  }
  router_wgrad_reduce_kernel<<<(E * H + 255) / 256, 256, 0, st>>>(partial, splits, E * H, H, dlc, dwg);
  count_launch();
}

void launch_grad_reduce_scatter(const PlanTables* pt, const PeerTable& peers, int E, int rank, long long S,
                                long long flat, float* grad_shard, cudaStream_t st) {
  grad_reduce_scatter_kernel<<<dim3(64, E), 256, 0, st>>>(pt, peers, E, rank, S, flat, grad_shard);
  count_launch();
}

void launch_pack_expert(const __nv_bfloat16* w1, const __nv_bfloat16* w3, const __nv_bfloat16* w2, int H, int F,
                        __nv_bfloat16* flat, cudaStream_t st) {
  pack_expert_kernel<<<1024, 256, 0, st>>>(w1, w3, w2, H, F, flat);
  count_launch();
}

void launch_unpack_grad(const float* chunk, long long lo, long long hi, int H, int F, float* dw1, float* dw3,
                        float* dw2, cudaStream_t st) {
  unpack_grad_kernel<<<1024, 256, 0, st>>>(chunk, lo, hi, H, F, dw1, dw3, dw2);
  count_launch();
}

}  // namespace fsep

namespace fsep {
void launch_grad_rs_sum(const PlanTables* pt, const float* grad_full, const float* stage, int E, int N, int rank,
                        long long S, long long flat, float* grad_shard, cudaStream_t st) {
  grad_rs_sum_kernel<<<dim3(std::max(1, 2 * 148 * 8 / E), E), 256, 0, st>>>(pt, grad_full, stage, N, rank, S, flat, grad_shard);
  count_launch();
}
}  // namespace fsep
