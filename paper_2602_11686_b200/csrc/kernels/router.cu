// Router of the FSEP layer step: logits = x . wg^T (+ bias), top-k (ties to the
// lowest expert id), softmax over the selected k, per-block expert histograms and
// in-block slot ranks (token order).  CUDA cores, register-tiled.
//
// Canonical fp32 order (the bit-exactness contract with oracle/layer_oracle.py):
//   logit[t][e] = fma(x[t][H-1], w[e][H-1], ... fma(x[t][1], w[e][1], fma(x[t][0], w[e][0], 0)) ...) + bias[t][e]
// i.e. one sequential fp32 accumulation over h.  Both operands are bf16, so each
// product is exact in fp32 and the FMA equals multiply-then-add; only the adds
// round, in a fixed order.  Tensor cores are not used here on purpose: their
// accumulation order is not specified, and routing must be reproducible bit for
// bit on the CPU.
//
// Block = kBlockTokens (64) tokens x all E experts.  The hidden dimension is
// streamed in 64-wide chunks staged (bf16 -> fp32, transposed h-major) in shared
// memory; each thread owns a TT x TE (tokens x experts) register tile.  Staging
// reads whole 128-B row pieces per 8 lanes (coalesced); the transposed stores are
// XOR-swizzled by the h octet so they stay bank-conflict free.
#include <cuda_bf16.h>

#include <cfloat>
#include <cstdlib>
#include <string>
#include <stdexcept>

#include "kernels/fsep_types.cuh"
#include "kernels/kernels.hpp"
#include "kernels/routing.hpp"

namespace fsep {
namespace {

constexpr int kHC = 64;  // hidden chunk

__device__ __forceinline__ float2 ffma2_rn(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}


template <int TT, int TE>
__global__ void __launch_bounds__(512) router_gemm_kernel(const __nv_bfloat16* __restrict__ x,
                                                          const __nv_bfloat16* __restrict__ wg,
                                                          const float* __restrict__ bias, int T, int H, int E, int K,
                                                          int* __restrict__ topk_idx, float* __restrict__ topk_w,
                                                          int* __restrict__ intra_rank, int* __restrict__ blk_hist) {
  constexpr int BT = kBlockTokens;
  constexpr int kWords = BT / 32;
  extern __shared__ float smem[];
  // column c of row h lives at c ^ swz(h) (swz keeps 4-column groups aligned)
  const int EW = (E + 31) & ~31;    // 32-aligned row stride of the weight tile
  float* s_x = smem;                // [kHC][BT]    h-major, swizzled
  float* s_w = smem + kHC * BT;     // [kHC][EW]    h-major, swizzled
  float* s_logit = smem;            // [BT][E + 1]  (reuses the staging area afterwards)
  __shared__ int s_idx[BT][8];
  __shared__ unsigned s_mask[kMaxExperts][kWords];

  const int tid = threadIdx.x, nthr = blockDim.x;
  const int t0 = blockIdx.x * BT;
  const int egroups = E / TE;
  // the block is rounded up to whole warps (the top-k below shuffles over full warps);
  // threads past the ntg x egroups tiles only stage and rank
  const bool tiled = tid < (BT / TT) * egroups;
  const int tg = tiled ? tid / egroups : 0, eg = tiled ? tid % egroups : 0;  // this thread's tile
  for (int i = tid; i < kMaxExperts * kWords; i += nthr) (&s_mask[0][0])[i] = 0u;

  float acc[TT][TE];
#pragma unroll
  for (int i = 0; i < TT; ++i)
#pragma unroll
    for (int j = 0; j < TE; ++j) acc[i][j] = 0.f;

  // staging work items: x = BT tokens x 8 sixteen-byte pieces; w = E x 8 pieces.
  // Eight consecutive items are the eight pieces of one row (one 128-B line).
  const int x_items = BT * (kHC / 8), w_items = E * (kHC / 8);
  for (int h0 = 0; h0 < H; h0 += kHC) {
    __syncthreads();
    for (int it = tid; it < x_items; it += nthr) {
      const int tt = it >> 3, piece = it & 7;
      const int t = min(t0 + tt, T - 1);  // clamp: rows past T are never selected
      const uint4 q = __ldg(reinterpret_cast<const uint4*>(x + static_cast<size_t>(t) * H + h0) + piece);
      const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&q);
      const int col = tt ^ (piece << 2);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = __bfloat1622float2(b[k]);
        s_x[(piece * 8 + 2 * k) * BT + col] = f.x;
        s_x[(piece * 8 + 2 * k + 1) * BT + col] = f.y;
      }
    }
    for (int it = tid; it < w_items; it += nthr) {
      const int e = it >> 3, piece = it & 7;
      const uint4 q = __ldg(reinterpret_cast<const uint4*>(wg + static_cast<size_t>(e) * H + h0) + piece);
      const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&q);
      const int col = e ^ (piece << 2);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 f = __bfloat1622float2(b[k]);
        s_w[(piece * 8 + 2 * k) * EW + col] = f.x;
        s_w[(piece * 8 + 2 * k + 1) * EW + col] = f.y;
      }
    }
    __syncthreads();
    static_assert(TT % 4 == 0 && TE % 4 == 0, "register tile must be float4-aligned");
#pragma unroll 1
    for (int hb = 0; hb < kHC / 8; ++hb) {
      // one h octet shares its swizzle: hoist the tile addresses, then immediate offsets
      const int swz = hb << 2;
      const float* xo = s_x + hb * 8 * BT;
      const float* wo = s_w + hb * 8 * EW;
      int xc[TT / 4], wc[TE / 4];
#pragma unroll
      for (int i = 0; i < TT / 4; ++i) xc[i] = (tg * TT + 4 * i) ^ swz;
#pragma unroll
      for (int j = 0; j < TE / 4; ++j) wc[j] = (eg * TE + 4 * j) ^ swz;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      float xv[TT], wv[TE];
#pragma unroll
      for (int i = 0; i < TT; i += 4) {
        const float4 v = *reinterpret_cast<const float4*>(xo + u * BT + xc[i / 4]);
        xv[i] = v.x, xv[i + 1] = v.y, xv[i + 2] = v.z, xv[i + 3] = v.w;
      }
#pragma unroll
      for (int j = 0; j < TE; j += 4) {
        const float4 v = *reinterpret_cast<const float4*>(wo + u * EW + wc[j / 4]);
        wv[j] = v.x, wv[j + 1] = v.y, wv[j + 2] = v.z, wv[j + 3] = v.w;
      }
#pragma unroll
      for (int i = 0; i < TT; ++i)
#pragma unroll
        for (int j = 0; j < TE; j += 2) {  // FFMA2: two independent chains per instruction
          const float2 r = ffma2_rn(make_float2(xv[i], xv[i]), make_float2(wv[j], wv[j + 1]),
                                    make_float2(acc[i][j], acc[i][j + 1]));
          acc[i][j] = r.x;
          acc[i][j + 1] = r.y;
        }
    }
    }
  }
  __syncthreads();
  // logits (+ bias) -> shared memory
  if (tiled)
#pragma unroll
  for (int i = 0; i < TT; ++i) {
    const int tt = tg * TT + i;
    const int t = t0 + tt;
#pragma unroll
    for (int j = 0; j < TE; ++j) {
      const int e = eg * TE + j;
      float v = acc[i][j];
      if (bias && t < T) v = __fadd_rn(v, __ldg(bias + static_cast<size_t>(t) * E + e));
      s_logit[tt * (E + 1) + e] = v;
    }
  }
  __syncthreads();
  // top-k per token: a warp per token (largest logit, lowest id on ties)
  const int warp = tid >> 5, lane = tid & 31, nwarps = nthr >> 5;
  for (int tt = warp; tt < BT; tt += nwarps) {
    const int t = t0 + tt;
    if (t >= T) break;
    float mine[kMaxExperts / 32];
#pragma unroll
    for (int q = 0; q < kMaxExperts / 32; ++q) {
      const int e = q * 32 + lane;
      mine[q] = e < E ? s_logit[tt * (E + 1) + e] : -FLT_MAX;
    }
    float sel_v[8];
    int sel_e[8];
    for (int k = 0; k < K; ++k) {
      float bv = -FLT_MAX;
      int be = 0x7fffffff;
#pragma unroll
      for (int q = 0; q < kMaxExperts / 32; ++q) {
        const int e = q * 32 + lane;
        if (e < E && (mine[q] > bv || (mine[q] == bv && e < be))) {
          bv = mine[q];
          be = e;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oe = __shfl_xor_sync(0xffffffffu, be, o);
        if (ov > bv || (ov == bv && oe < be)) {
          bv = ov;
          be = oe;
        }
      }
      sel_v[k] = bv;
      sel_e[k] = be;
#pragma unroll
      for (int q = 0; q < kMaxExperts / 32; ++q)  // exclude the winner (below -FLT_MAX)
        if (q == (be >> 5) && (be & 31) == lane) mine[q] = -INFINITY;
    }
    if (lane == 0) {
      float w[8], s = 0.f;
      for (int k = 0; k < K; ++k) {
        w[k] = expf(sel_v[k] - sel_v[0]);
        s += w[k];
      }
      for (int k = 0; k < K; ++k) {
        topk_idx[static_cast<size_t>(t) * K + k] = sel_e[k];
        topk_w[static_cast<size_t>(t) * K + k] = w[k] / s;
        s_idx[tt][k] = sel_e[k];
        atomicOr(&s_mask[sel_e[k]][tt >> 5], 1u << (tt & 31));
      }
    }
  }
  __syncthreads();
  // per-slot rank within the block (tokens with the same expert before me) + counts
  for (int tt = tid; tt < BT; tt += nthr) {
    const int t = t0 + tt;
    if (t >= T) break;
    const int w = tt >> 5, l = tt & 31;
    for (int k = 0; k < K; ++k) {
      const int e = s_idx[tt][k];
      int r = __popc(s_mask[e][w] & ((1u << l) - 1u));
      for (int ww = 0; ww < w; ++ww) r += __popc(s_mask[e][ww]);
      intra_rank[static_cast<size_t>(t) * K + k] = r;
    }
  }
  for (int e = tid; e < E; e += nthr) {
    int cnt = 0;
#pragma unroll
    for (int w = 0; w < kWords; ++w) cnt += __popc(s_mask[e][w]);
    blk_hist[static_cast<size_t>(blockIdx.x) * E + e] = cnt;
  }
}

// Small-E variant (E <= 16): one thread per token holds all E accumulators and
// streams its token row from HBM in 16-byte pieces; expert-weight pieces are the
// same for every thread of the warp (broadcast loads, L1-resident).  Same
// canonical order: per (token, expert) one FMA chain over h ascending.
template <int E_>
__global__ void __launch_bounds__(kBlockTokens) router_small_kernel(
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ wg, const float* __restrict__ bias, int T,
    int H, int K, int* __restrict__ topk_idx, float* __restrict__ topk_w, int* __restrict__ intra_rank,
    int* __restrict__ blk_hist) {
  constexpr int BT = kBlockTokens;
  constexpr int kWords = BT / 32;
  __shared__ int s_idx[BT][8];
  __shared__ unsigned s_mask[E_][kWords];
  extern __shared__ uint4 s_w4[];  // the whole router weight [E_][H] bf16 (64 KB for E=8, H=4096)
  const int tt = threadIdx.x;
  const int t = blockIdx.x * BT + tt;
  const int pieces = H / 8;
  for (int i = tt; i < E_ * kWords; i += BT) (&s_mask[0][0])[i] = 0u;
  for (int i = tt; i < E_ * pieces; i += BT) s_w4[i] = __ldg(reinterpret_cast<const uint4*>(wg) + i);
  __syncthreads();
  if (t < T) {
    float acc[E_];
#pragma unroll
    for (int e = 0; e < E_; ++e) acc[e] = 0.f;
    const uint4* xr = reinterpret_cast<const uint4*>(x + static_cast<size_t>(t) * H);
    // 8-deep register prefetch ring over the token row: each thread streams its
    // own row, so memory-level parallelism has to come from the ring, not from
    // the (few) resident warps.
    constexpr int D = 8;
    uint4 ring[D];
#pragma unroll
    for (int i = 0; i < D; ++i) ring[i] = __ldg(xr + i);
    for (int p0 = 0; p0 < pieces; p0 += D) {
      uint4 cur[D];
#pragma unroll
      for (int i = 0; i < D; ++i) cur[i] = ring[i];
      if (p0 + D < pieces) {
#pragma unroll
        for (int i = 0; i < D; ++i) ring[i] = __ldg(xr + p0 + D + i);
      }
#pragma unroll
      for (int i = 0; i < D; ++i) {
      const int p = p0 + i;
      float xf[8];
      {
        const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&cur[i]);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f = __bfloat1622float2(b[k]);
          xf[2 * k] = f.x;
          xf[2 * k + 1] = f.y;
        }
      }
#pragma unroll
      for (int e = 0; e < E_; ++e) {
        const uint4 q = s_w4[e * pieces + p];
        const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 f = __bfloat1622float2(b[k]);
          acc[e] = __fmaf_rn(xf[2 * k], f.x, acc[e]);
          acc[e] = __fmaf_rn(xf[2 * k + 1], f.y, acc[e]);
        }
      }
      }
    }
    if (bias) {
#pragma unroll
      for (int e = 0; e < E_; ++e) acc[e] = __fadd_rn(acc[e], __ldg(bias + static_cast<size_t>(t) * E_ + e));
    }
    // top-k: largest logit, lowest id on ties (strict > in ascending e)
    unsigned taken = 0u;
    float sel_v[8];
    int sel_e[8];
    for (int k = 0; k < K; ++k) {
      float bv = -INFINITY;
      int be = -1;
#pragma unroll
      for (int e = 0; e < E_; ++e)
        if (!(taken >> e & 1u) && (be < 0 || acc[e] > bv)) {
          bv = acc[e];
          be = e;
        }
      taken |= 1u << be;
      sel_v[k] = bv;
      sel_e[k] = be;
    }
    float w[8], s = 0.f;
    for (int k = 0; k < K; ++k) {
      w[k] = expf(sel_v[k] - sel_v[0]);
      s += w[k];
    }
    for (int k = 0; k < K; ++k) {
      topk_idx[static_cast<size_t>(t) * K + k] = sel_e[k];
      topk_w[static_cast<size_t>(t) * K + k] = w[k] / s;
      s_idx[tt][k] = sel_e[k];
      atomicOr(&s_mask[sel_e[k]][tt >> 5], 1u << (tt & 31));
    }
  }
  __syncthreads();
  if (t < T) {
    const int w = tt >> 5, l = tt & 31;
    for (int k = 0; k < K; ++k) {
      const int e = s_idx[tt][k];
      int r = __popc(s_mask[e][w] & ((1u << l) - 1u));
      for (int ww = 0; ww < w; ++ww) r += __popc(s_mask[e][ww]);
      intra_rank[static_cast<size_t>(t) * K + k] = r;
    }
  }
  for (int e = tt; e < E_; e += BT) {
    int cnt = 0;
#pragma unroll
    for (int w = 0; w < kWords; ++w) cnt += __popc(s_mask[e][w]);
    blk_hist[static_cast<size_t>(blockIdx.x) * E_ + e] = cnt;
  }
}

// Small-E variant, packed: E_/2 threads per token, each owning the FMA chains of
// two experts (e0, e0+1) and advancing both with one fma.rn.f32x2 (FFMA2: two
// independent IEEE fp32 FMAs, so each chain keeps the canonical order).  The
// router weight sits in shared memory h-major ([H][E_] bf16) so a thread's pair
// of weights for one h is a single 32-bit load; the token row streams from HBM
// through a register ring (threads of one token read the same addresses).
template <int E_>
__global__ void __launch_bounds__(kBlockTokens * E_ / 2) router_pair_kernel(
    const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ wg, const float* __restrict__ bias, int T,
    int H, int K, int* __restrict__ topk_idx, float* __restrict__ topk_w, int* __restrict__ intra_rank,
    int* __restrict__ blk_hist) {
  constexpr int BT = kBlockTokens, EP = E_ / 2, NT = BT * EP;
  constexpr int kWords = BT / 32;
  __shared__ int s_idx[BT][8];
  __shared__ unsigned s_mask[E_][kWords];
  __shared__ float s_logit[BT][E_ + 1];
  extern __shared__ __nv_bfloat162 s_wt[];  // [H][E_/2] pairs: s_wt[h*EP + p] = (w[2p][h], w[2p+1][h])
  const int tid = threadIdx.x;
  const int tt = tid / EP, ep = tid % EP;
  const int t = blockIdx.x * BT + tt;
  for (int i = tid; i < E_ * kWords; i += NT) (&s_mask[0][0])[i] = 0u;
  for (int i = tid; i < H * EP; i += NT) {  // transpose the router weight into h-major pairs
    const int h = i / EP, p = i % EP;
    s_wt[i] = __halves2bfloat162(wg[static_cast<size_t>(2 * p) * H + h], wg[static_cast<size_t>(2 * p + 1) * H + h]);
  }
  __syncthreads();
  float2 acc = make_float2(0.f, 0.f);
  const uint4* xr = reinterpret_cast<const uint4*>(x + static_cast<size_t>(min(t, T - 1)) * H);
  const int pieces = H / 8;
  constexpr int D = 8;
  uint4 ring[D];
#pragma unroll
  for (int i = 0; i < D; ++i) ring[i] = __ldg(xr + i);
  for (int p0 = 0; p0 < pieces; p0 += D) {
    uint4 cur[D];
#pragma unroll
    for (int i = 0; i < D; ++i) cur[i] = ring[i];
    if (p0 + D < pieces) {
#pragma unroll
      for (int i = 0; i < D; ++i) ring[i] = __ldg(xr + p0 + D + i);
    }
#pragma unroll
    for (int i = 0; i < D; ++i) {
      const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&cur[i]);
      const __nv_bfloat162* wp = s_wt + static_cast<size_t>(p0 + i) * 8 * EP + ep;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 xf = __bfloat1622float2(b[k]);
        const float2 w0 = __bfloat1622float2(wp[(2 * k) * EP]);
        const float2 w1 = __bfloat1622float2(wp[(2 * k + 1) * EP]);
        acc = ffma2_rn(make_float2(xf.x, xf.x), w0, acc);
        acc = ffma2_rn(make_float2(xf.y, xf.y), w1, acc);
      }
    }
  }
  if (t < T) {
    float a0 = acc.x, a1 = acc.y;
    if (bias) {
      a0 = __fadd_rn(a0, __ldg(bias + static_cast<size_t>(t) * E_ + 2 * ep));
      a1 = __fadd_rn(a1, __ldg(bias + static_cast<size_t>(t) * E_ + 2 * ep + 1));
    }
    s_logit[tt][2 * ep] = a0;
    s_logit[tt][2 * ep + 1] = a1;
  }
  __syncthreads();
  if (tid < BT && blockIdx.x * BT + tid < T) {  // top-k per token (same rule as router_small_kernel)
    const int u = tid, tu = blockIdx.x * BT + tid;
    unsigned taken = 0u;
    float sel_v[8];
    int sel_e[8];
    for (int k = 0; k < K; ++k) {
      float bv = -INFINITY;
      int be = -1;
#pragma unroll
      for (int e = 0; e < E_; ++e)
        if (!(taken >> e & 1u) && (be < 0 || s_logit[u][e] > bv)) {
          bv = s_logit[u][e];
          be = e;
        }
      taken |= 1u << be;
      sel_v[k] = bv;
      sel_e[k] = be;
    }
    float w[8], sum = 0.f;
    for (int k = 0; k < K; ++k) {
      w[k] = expf(sel_v[k] - sel_v[0]);
      sum += w[k];
    }
    for (int k = 0; k < K; ++k) {
      topk_idx[static_cast<size_t>(tu) * K + k] = sel_e[k];
      topk_w[static_cast<size_t>(tu) * K + k] = w[k] / sum;
      s_idx[u][k] = sel_e[k];
      atomicOr(&s_mask[sel_e[k]][u >> 5], 1u << (u & 31));
    }
  }
  __syncthreads();
  if (tid < BT && blockIdx.x * BT + tid < T) {
    const int u = tid, tu = blockIdx.x * BT + tid;
    const int w = u >> 5, l = u & 31;
    for (int k = 0; k < K; ++k) {
      const int e = s_idx[u][k];
      int r = __popc(s_mask[e][w] & ((1u << l) - 1u));
      for (int ww = 0; ww < w; ++ww) r += __popc(s_mask[e][ww]);
      intra_rank[static_cast<size_t>(tu) * K + k] = r;
    }
  }
  for (int e = tid; e < E_; e += NT) {
    int cnt = 0;
#pragma unroll
    for (int w = 0; w < kWords; ++w) cnt += __popc(s_mask[e][w]);
    blk_hist[static_cast<size_t>(blockIdx.x) * E_ + e] = cnt;
  }
}

template <int TT, int TE>
void launch_tiled(const RouterArgs& a, int nblk, cudaStream_t st) {
  const int threads = ((kBlockTokens / TT) * (a.E / TE) + 31) & ~31;
  const size_t smem = static_cast<size_t>(kHC) * (kBlockTokens + ((a.E + 31) & ~31)) * sizeof(float);
  set_smem_attr(reinterpret_cast<const void*>(router_gemm_kernel<TT, TE>), 96 * 1024);
  router_gemm_kernel<TT, TE><<<nblk, threads, smem, st>>>(a.x, a.wg, a.bias, a.T, a.H, a.E, a.K, a.topk_idx,
                                                          a.topk_w, a.intra_rank, a.blk_hist);
}

}  // namespace

void launch_router(const RouterArgs& a, cudaStream_t st) {
  const int nblk = (a.T + kBlockTokens - 1) / kBlockTokens;
  if (nblk == 0) return;
  if (a.E % 8 != 0 || a.E > kMaxExperts) throw std::runtime_error("router: n_experts must be a multiple of 8, <= 256");
  if (a.H % kHC != 0) throw std::runtime_error("router: hidden must be a multiple of 64");
  const size_t w_bytes = static_cast<size_t>(a.E) * a.H * sizeof(__nv_bfloat16);
  set_smem_attr(reinterpret_cast<const void*>(router_small_kernel<8>), 200 * 1024);
  set_smem_attr(reinterpret_cast<const void*>(router_small_kernel<16>), 200 * 1024);
  static const bool small = [] {
    const char* v = std::getenv("FSEP_ROUTER");
    return v && std::string(v) == "small";
  }();
  set_smem_attr(reinterpret_cast<const void*>(router_pair_kernel<8>), 200 * 1024);
  set_smem_attr(reinterpret_cast<const void*>(router_pair_kernel<16>), 200 * 1024);
  if (!small && a.E == 8 && w_bytes <= 200 * 1024)
    router_pair_kernel<8><<<nblk, kBlockTokens * 4, w_bytes, st>>>(a.x, a.wg, a.bias, a.T, a.H, a.K, a.topk_idx,
                                                                   a.topk_w, a.intra_rank, a.blk_hist);
  else if (!small && a.E == 16 && w_bytes <= 200 * 1024)
    router_pair_kernel<16><<<nblk, kBlockTokens * 8, w_bytes, st>>>(a.x, a.wg, a.bias, a.T, a.H, a.K, a.topk_idx,
                                                                    a.topk_w, a.intra_rank, a.blk_hist);
  else if (a.E == 8 && w_bytes <= 200 * 1024)
    router_small_kernel<8><<<nblk, kBlockTokens, w_bytes, st>>>(a.x, a.wg, a.bias, a.T, a.H, a.K, a.topk_idx,
                                                               a.topk_w, a.intra_rank, a.blk_hist);
  else if (a.E == 16 && w_bytes <= 200 * 1024)
    router_small_kernel<16><<<nblk, kBlockTokens, w_bytes, st>>>(a.x, a.wg, a.bias, a.T, a.H, a.K, a.topk_idx,
                                                                a.topk_w, a.intra_rank, a.blk_hist);
  else
  {
    static const int tile = [] {
      const char* v = std::getenv("FSEP_ROUTER_TILE");
      return v ? std::atoi(v) : 4;  // 8x8 tiles measured slower (0.66 vs 0.57 ms, fine config)
    }();
    if (tile == 8 && a.E % 8 == 0)
      launch_tiled<8, 8>(a, nblk, st);  // 8 x E/8 threads, 8x8 register tiles (half the smem traffic per FMA)
    else if (a.E > 128 || tile == 84)
      launch_tiled<8, 4>(a, nblk, st);  // 8 x E/4 threads (<= 512 for E <= 256)
    else
      launch_tiled<4, 4>(a, nblk, st);  // 16 x E/4 threads
  }
  count_launch();
}

}  // namespace fsep
