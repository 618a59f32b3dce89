// Grouped expert GEMM for the FSEP layer step on sm_100a: tcgen05.mma with
// fp32 accumulators in TMEM, operands staged by TMA (SWIZZLE_128B) through a
// 4-stage mbarrier ring, warp-specialised and persistent (one CTA per SM).
//
//   warp 0      TMA producer (one elected lane)
//   warp 1      TMEM allocator + MMA issuer (one elected lane)
//   warps 2..5  epilogue: TMEM -> registers -> fused op -> global
//
// Tile 128 x 256 x 64 (UMMA 128x256x16, cta_group::1).  The accumulator is
// double-buffered in TMEM (2 x 256 of the 512 columns) so the epilogue of tile i
// overlaps the MMAs of tile i+1.
//
// Two grouping modes, both driven by device-side per-group row counts (no host
// sync -- the routing kernels write them):
//   M-grouped (kGroupK=false): C_g[rows_g, N] = A[rows of g, K] * B_g[N, K]^T.
//       A is the dispatched-token buffer (expert-major, each group padded to
//       128 rows); B_g the restored weights of local expert slot g (3-D map).
//   K-grouped (kGroupK=true):  C_g[M, N] = A_g[rows_g, M]^T * B_g[rows_g, N]
//       (weight gradients: the ragged token dimension is the reduction).
// Operand majorness is a template parameter (K-major or MN-major for A and B),
// so dgrad/wgrad read activations and weights in place, without transposes.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "kernels/fsep_types.cuh"
#include "kernels/sm100_ptx.cuh"

namespace fsep {

enum Epi : int {
  kEpiBf16 = 0,       // out[row, n] = bf16(acc)
  kEpiSwigluFwd = 1,  // acc tile = [gate 128 | up 128] -> h (bf16, 256 cols) and act = silu(g)*u (128 cols)
  kEpiSwigluBwd = 2,  // acc = dAct tile (256 f cols); reads h, writes dH = [dgate | dup] interleaved
  kEpiF32 = 3,        // out_g[m, n] = acc (fp32 weight gradient)
};

struct GemmParams {
  int num_groups;
  const int* group_rows;  // [G] padded rows per group (multiple of 128)
  const int* group_off;   // [G] first row of group g in the row-indexed operands
  int M, N, K;            // fixed dims (M: K-grouped only; K: M-grouped only)
  void* out;
  long long ldo;
  long long out_group_stride;  // K-grouped: elements between group outputs
  void* out2;                  // SwigluFwd: act
  long long ldo2;
  const void* aux;  // SwigluBwd: h
  long long ld_aux;
  int policy;  // L2 hints: bits 0-1 A, bits 2-3 B (0 default for the mode, 1 normal, 2 evict_first, 3 evict_last);
               // bit 8: pair kernel runs a <=128-column last N tile at full N=256 (no N=128 tail MMA)
               // bit 9: pair kernel uses a plain round-robin tile schedule (no snake / LPT group order)
               // bit 10: pair kernel releases the TMEM accumulator with a cluster-scope release (A/B)
               // bit 11: no wave synchronisation for this launch (A/B; launcher-side)
               // bit 12: no M=128 tail tiles (masked M=256 tiles instead; A/B)
               // bit 13: the launch has a 64-row-box B map (gate-up M=128 tail tiles)
               // bit 14: odd waves load their k-blocks in reverse order (L2 reuse across waves; A/B)
               // bit 15: no L2 prefetch of h in the SwiGLU' epilogue (A/B)
  int raster;  // tile order within a group: 0 mode default, 1 m-inner, 2 n-inner, 3+ = m-chunks of `raster` tiles, n-inner
  // Optional per-group readiness (M-grouped only): before loading B of group g the
  // producer waits until ready[g * ready_n + q] has reached ready_epoch for all
  // q < ready_n (restored expert chunks landing from the copy engines).
  const unsigned* ready;
  unsigned ready_epoch;
  int ready_n;
  // Bounded wait: after ready_timeout_ns without the flag the producer raises
  // kErrRestoreTimeout in err (host-mapped) and stops waiting for the launch.
  unsigned* err;
  unsigned long long ready_timeout_ns;
  // Optional row scatter (kEpiBf16, M-grouped): output row r is stored to
  // scatter[code >> 26] + (code & 0x3FFFFFF) * ldo, code = row_src[r] (code < 0:
  // padding row, not stored).  This is how the expert outputs travel straight
  // from the GEMM epilogue into the token owner's slot rows over NVLink.
  const int* row_src;
  __nv_bfloat16* const* scatter;
  long long scatter_rows;
  // Optional wave synchronisation (pair kernel, M-grouped): before loading the tiles
  // of wave w every CTA's producer waits (bounded) until all CTAs with a tile in
  // wave w have issued the loads of wave w-1, so the CTAs stream the shared A / B
  // panels along K in step and the panels are fetched from DRAM once per wave.
  // wave_sync[w] are arrival counters, zeroed before the launch.
  int* wave_sync;
};

__device__ __forceinline__ __nv_bfloat16* bf16_out_row(const GemmParams& p, long long row) {
  if (p.row_src == nullptr) return static_cast<__nv_bfloat16*>(p.out) + row * p.ldo;
  const int code = p.row_src[row];
  if (code < 0) return nullptr;
  const long long idx = code & 0x3FFFFFF;
  if (idx >= p.scatter_rows) return nullptr;
  return p.scatter[code >> 26] + idx * p.ldo;
}

// The flags are written by the pushing peers' copy engines (another GPU in real
// mode): system-scope acquire.  Returns false after a timeout (error raised).
__device__ __forceinline__ bool wait_group_ready(const GemmParams& p, int g) {
  if (p.ready == nullptr) return true;
  const unsigned long long t0 = globaltimer_ns();
  for (int q = 0; q < p.ready_n; ++q) {
    const unsigned* f = p.ready + g * p.ready_n + q;
    while (true) {
      unsigned v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
      if (static_cast<int>(v - p.ready_epoch) >= 0) break;
      if (globaltimer_ns() - t0 > p.ready_timeout_ns) {
        raise_err(p.err, kErrRestoreTimeout);
        return false;
      }
      __nanosleep(256);
    }
  }
  // the chunks were written by copy engines (generic proxy); TMA reads via the async proxy
  asm volatile("fence.proxy.async.global;" ::: "memory");
  return true;
}

// Returns false on timeout (~0.4 ms: the CTAs are not all co-resident, e.g. another
// kernel holds SMs); the caller then stops synchronising for the rest of the launch.
__device__ __forceinline__ bool wave_barrier(int* ctr, int expected) {
  atomicAdd(ctr, 1);
  for (int spin = 0; spin < 4000; ++spin) {
    int v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    if (v >= expected) return true;
    __nanosleep(64);
  }
  return false;
}

namespace gemm {
constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;  // 16 KB
constexpr int B_BYTES = BN * BK * 2;  // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int MAX_GROUPS = 256;
constexpr int THREADS = 192;
constexpr int SMEM_BYTES = 1024 /*align slack*/ + STAGES * STAGE_BYTES + 256 /*barriers*/ + (MAX_GROUPS + 1) * 4;
}  // namespace gemm

// MUFU-based (approximate reciprocal, ~2 ulp fp32): the result is rounded to bf16, and an
// IEEE division would cost a slow-path subroutine call per element in the epilogue.
#ifdef FSEP_SIGMOID_TANH
// A/B variant: one MUFU op (tanh.approx) instead of two (ex2 + rcp); absolute error ~2^-12.
__device__ __forceinline__ float sigmoid_f(float g) {
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.5f * g));
  return fmaf(0.5f, t, 0.5f);
}
#else
__device__ __forceinline__ float sigmoid_f(float g) { return __fdividef(1.0f, 1.0f + __expf(-g)); }
#endif
__device__ __forceinline__ float silu_f(float g) { return g * sigmoid_f(g); }

__device__ __forceinline__ uint64_t pick_policy(int code, bool first_by_default) {
  switch (code) {
    case 1: {
      uint64_t p;
      asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
      return p;
    }
    case 2: return ptx::policy_evict_first();
    case 3: return ptx::policy_evict_last();
    default: return first_by_default ? ptx::policy_evict_first() : ptx::policy_evict_last();
  }
}

// Tile order inside one group of mb_count x nb_count output tiles.
__device__ __forceinline__ void raster_tile(int local, int mb_count, int nb_count, int raster, bool group_k, int& mb,
                                            int& nbk) {
  const int mode = raster == 0 ? (group_k ? 2 : 1) : raster;
  if (mode == 1) {
    mb = local % mb_count;
    nbk = local / mb_count;
  } else if (mode == 2) {
    nbk = local % nb_count;
    mb = local / nb_count;
  } else {  // chunks of `mode` m-tiles; inside a chunk m fastest, then n
    const int chunk = mode;
    const int per_chunk = chunk * nb_count;
    const int c = local / per_chunk;
    const int rem = local % per_chunk;
    const int rows_in_chunk = min(chunk, mb_count - c * chunk);
    mb = c * chunk + rem % rows_in_chunk;
    nbk = rem / rows_in_chunk;
  }
}

template <bool kAMN, bool kBMN, bool kGroupK, int kEpi>
__global__ void __launch_bounds__(gemm::THREADS, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const GemmParams p) {
  using namespace gemm;
  using namespace fsep::ptx;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  int* tile_start = reinterpret_cast<int*>(smem + STAGES * STAGE_BYTES + 256);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int G = p.num_groups;
  const int nb = (p.N + BN - 1) / BN;

  if (threadIdx.x == 0) {
    int acc = 0;
    for (int g = 0; g < G; ++g) {
      tile_start[g] = acc;
      const int rows = p.group_rows[g];
      acc += kGroupK ? (p.M / BM) * nb : ((rows + BM - 1) / BM) * nb;
    }
    tile_start[G] = acc;
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 4);
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total_tiles = tile_start[G];

  // tile -> (group, m block, n block)
  auto decode = [&](int t, int& g, int& mb, int& nbk) {
    g = 0;
    while (tile_start[g + 1] <= t) ++g;
    const int local = t - tile_start[g];
    if (kGroupK) {
      nbk = local % nb;
      mb = local / nb;
    } else {
      const int mbs = (p.group_rows[g] + BM - 1) / BM;
      mb = local % mbs;
      nbk = local / mbs;
    }
  };
  auto k_blocks = [&](int g) { return kGroupK ? p.group_rows[g] / BK : p.K / BK; };

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (elect_one()) {
      const uint64_t pol_a = kGroupK ? policy_evict_first() : policy_evict_last();
      const uint64_t pol_b = kGroupK ? policy_evict_last() : policy_evict_first();
      int s = 0;
      uint32_t ph = 0;
      int ready_g = -1;
      bool ready_live = true;
      for (int t = blockIdx.x; t < total_tiles; t += gridDim.x) {
        int g, mb, nbk;
        decode(t, g, mb, nbk);
        const int nk = k_blocks(g);
        const int row0 = p.group_off[g];
        if (!kGroupK && g != ready_g && ready_live) {
          ready_live = wait_group_ready(p, g);  // false: timed out (error raised), stop waiting
          ready_g = g;
        }
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&empty_bar[s], ph ^ 1);
          uint8_t* sA = smem + s * STAGE_BYTES;
          uint8_t* sB = sA + A_BYTES;
          mbar_arrive_expect_tx(&full_bar[s], STAGE_BYTES);
          if (!kAMN) {  // A[rows, K] K-major: one 64 x 128 box
            tma_load_2d(sA, &tmA, &full_bar[s], kb * BK, row0 + mb * BM, pol_a);
          } else {      // A[rows(K), M] MN-major: two 64(M) x 64(K) boxes
#pragma unroll
            for (int i = 0; i < BM / 64; ++i)
              tma_load_2d(sA + i * 8192, &tmA, &full_bar[s], mb * BM + i * 64, row0 + kb * BK, pol_a);
          }
          if (!kGroupK) {  // per-group weights: 3-D map (inner, outer, group)
            if (!kBMN) {
              tma_load_3d(sB, &tmB, &full_bar[s], kb * BK, nbk * BN, g, pol_b);
            } else {
#pragma unroll
              for (int i = 0; i < BN / 64; ++i)
                tma_load_3d(sB + i * 8192, &tmB, &full_bar[s], nbk * BN + i * 64, kb * BK, g, pol_b);
            }
          } else {  // B[rows(K), N] MN-major
#pragma unroll
            for (int i = 0; i < BN / 64; ++i)
              tma_load_2d(sB + i * 8192, &tmB, &full_bar[s], nbk * BN + i * 64, row0 + kb * BK, pol_b);
          }
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = ptx::idesc_bf16(BM, BN, kAMN, kBMN);
    int s = 0;
    uint32_t ph = 0;
    int it = 0;
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++it) {
      int g, mb, nbk;
      decode(t, g, mb, nbk);
      const int nk = k_blocks(g);
      const int as = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      mbar_wait(&tempty_bar[as], aph ^ 1);
      tc_fence_after();
      const uint32_t tmem_d = tmem_base + as * BN;
      if (nk == 0) {
        if (lane == 0) mbar_arrive(&tfull_bar[as]);
        __syncwarp();
        continue;
      }
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait(&full_bar[s], ph);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t a0 = smem_u32(smem + s * STAGE_BYTES);
          const uint32_t b0 = a0 + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = kAMN ? smem_desc(a0 + k * 2048, 8192, 1024) : smem_desc(a0 + k * 32, 16, 1024);
            const uint64_t bd = kBMN ? smem_desc(b0 + k * 2048, 8192, 1024) : smem_desc(b0 + k * 32, 16, 1024);
            umma_bf16(tmem_d, ad, bd, idesc, (kb | k) ? 1u : 0u);
          }
          umma_commit(&empty_bar[s]);
          if (kb == nk - 1) umma_commit(&tfull_bar[as]);
        }
        __syncwarp();
        if (++s == STAGES) {
          s = 0;
          ph ^= 1;
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const uint32_t quarter = warp & 3;           // TMEM lane quarter this warp may access
    const int r = static_cast<int>(quarter * 32 + lane);  // row within the tile
    int it = 0;
    for (int t = blockIdx.x; t < total_tiles; t += gridDim.x, ++it) {
      int g, mb, nbk;
      decode(t, g, mb, nbk);
      const int as = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      mbar_wait(&tfull_bar[as], aph);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((quarter * 32) << 16) + as * BN;
      const bool empty_k = k_blocks(g) == 0;
      if (kEpi == kEpiF32) {
        float* out = static_cast<float*>(p.out) + static_cast<long long>(g) * p.out_group_stride +
                     static_cast<long long>(mb * BM + r) * p.ldo;
#pragma unroll 1
        for (int j = 0; j < BN / 32; ++j) {
          const int col = nbk * BN + j * 32;
          if (col >= p.N) break;
          float v[32];
          if (empty_k) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.f;
          } else {
            tmem_ld32(taddr + j * 32, v);
          }
          float4* dst = reinterpret_cast<float4*>(out + col);
#pragma unroll
          for (int i = 0; i < 8; ++i) dst[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        }
      } else if (kEpi == kEpiBf16) {
        const long long row = p.group_off[g] + mb * BM + r;
        __nv_bfloat16* out = bf16_out_row(p, row);
#pragma unroll 1
        for (int j = 0; j < BN / 32; ++j) {
          const int col = nbk * BN + j * 32;
          if (col >= p.N) break;
          float v[32];
          tmem_ld32(taddr + j * 32, v);  // warp-collective: every lane loads, only live rows store
          if (out == nullptr) continue;
          uint4* dst = reinterpret_cast<uint4*>(out + col);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            dst[i] = make_uint4(pack_bf16(v[8 * i], v[8 * i + 1]), pack_bf16(v[8 * i + 2], v[8 * i + 3]),
                                pack_bf16(v[8 * i + 4], v[8 * i + 5]), pack_bf16(v[8 * i + 6], v[8 * i + 7]));
        }
      } else if (kEpi == kEpiSwigluFwd) {
        // Accumulator columns [0,128) = gate f in [f0, f0+128), [128,256) = up.
        const long long row = p.group_off[g] + mb * BM + r;
        __nv_bfloat16* h = static_cast<__nv_bfloat16*>(p.out) + row * p.ldo + nbk * BN;
        __nv_bfloat16* act = static_cast<__nv_bfloat16*>(p.out2) + row * p.ldo2 + nbk * (BN / 2);
#pragma unroll 1
        for (int j = 0; j < 4; ++j) {
          float gv[32], uv[32];
          tmem_ld32(taddr + j * 32, gv);
          tmem_ld32(taddr + 128 + j * 32, uv);
          uint4* hg = reinterpret_cast<uint4*>(h + j * 32);
          uint4* hu = reinterpret_cast<uint4*>(h + 128 + j * 32);
          uint4* ao = reinterpret_cast<uint4*>(act + j * 32);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            hg[i] = make_uint4(pack_bf16(gv[8 * i], gv[8 * i + 1]), pack_bf16(gv[8 * i + 2], gv[8 * i + 3]),
                               pack_bf16(gv[8 * i + 4], gv[8 * i + 5]), pack_bf16(gv[8 * i + 6], gv[8 * i + 7]));
            hu[i] = make_uint4(pack_bf16(uv[8 * i], uv[8 * i + 1]), pack_bf16(uv[8 * i + 2], uv[8 * i + 3]),
                               pack_bf16(uv[8 * i + 4], uv[8 * i + 5]), pack_bf16(uv[8 * i + 6], uv[8 * i + 7]));
            float a[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) a[q] = silu_f(gv[8 * i + q]) * uv[8 * i + q];
            ao[i] = make_uint4(pack_bf16(a[0], a[1]), pack_bf16(a[2], a[3]), pack_bf16(a[4], a[5]),
                               pack_bf16(a[6], a[7]));
          }
        }
      } else {  // kEpiSwigluBwd
        const long long row = p.group_off[g] + mb * BM + r;
        const __nv_bfloat16* h = static_cast<const __nv_bfloat16*>(p.aux) + row * p.ld_aux;
        __nv_bfloat16* dh = static_cast<__nv_bfloat16*>(p.out) + row * p.ldo;
#pragma unroll 1
        for (int j = 0; j < BN / 32; ++j) {
          const int f = nbk * BN + j * 32;
          if (f >= p.N) break;
          const int hcol = (f / 128) * 256 + (f % 128);
          float da[32];
          tmem_ld32(taddr + j * 32, da);
          const uint4* hg4 = reinterpret_cast<const uint4*>(h + hcol);
          const uint4* hu4 = reinterpret_cast<const uint4*>(h + hcol + 128);
          uint4* dg4 = reinterpret_cast<uint4*>(dh + hcol);
          uint4* du4 = reinterpret_cast<uint4*>(dh + hcol + 128);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const uint4 gq = hg4[i], uq = hu4[i];
            const __nv_bfloat16* gb = reinterpret_cast<const __nv_bfloat16*>(&gq);
            const __nv_bfloat16* ub = reinterpret_cast<const __nv_bfloat16*>(&uq);
            float dg[8], du[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              const float gg = __bfloat162float(gb[q]);
              const float uu = __bfloat162float(ub[q]);
              const float sg = sigmoid_f(gg);
              const float d = da[8 * i + q];
              du[q] = d * gg * sg;
              dg[q] = d * uu * sg * (1.0f + gg * (1.0f - sg));
            }
            dg4[i] = make_uint4(pack_bf16(dg[0], dg[1]), pack_bf16(dg[2], dg[3]), pack_bf16(dg[4], dg[5]),
                                pack_bf16(dg[6], dg[7]));
            du4[i] = make_uint4(pack_bf16(du[0], du[1]), pack_bf16(du[2], du[3]), pack_bf16(du[4], du[5]),
                                pack_bf16(du[6], du[7]));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[as]);
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem_base);
  }
}

}  // namespace fsep
