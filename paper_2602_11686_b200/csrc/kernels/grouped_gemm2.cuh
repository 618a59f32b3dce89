// Grouped expert GEMM, CTA-pair version (tcgen05 cta_group::2) -- the
// production kernel of the FSEP layer step on sm_100a.
//
// A cluster of 2 CTAs (one TPC) computes a 256 x 256 output tile with
// UMMA 256x256x16: each CTA stages its 128 rows of A and its 128 columns of B
// (TMA, SWIZZLE_128B), so per-SM shared-memory traffic per FLOP is 2/3 of the
// 128x256 single-CTA tile and a 6-stage ring (32 KB/stage/CTA) gives 1.5x the
// latency cover.  The leader CTA issues the MMAs; tcgen05.commit multicasts
// stage-release and accumulator-ready to both CTAs; both CTAs' epilogues drain
// their own TMEM rows and release the accumulator to the leader.
//
//   warp 0      TMA producer (each CTA loads its halves; bytes land on CTA 0's barrier)
//   warp 1      TMEM allocator (cta_group::2) + MMA issuer (leader CTA)
//   warps 2..9  epilogue: 8 warps = 4 TMEM lane quarters x 2 column halves
//
// Grouping modes and operand majorness are as in grouped_gemm.cuh.  M-grouped
// segments are padded to 128 rows.  A group's last 256-row tile with only 128 rows
// left runs as an M=128 pair MMA ("tail tile"): each CTA stages 64 rows of A and the
// accumulator occupies N/2 TMEM columns -- lanes 0-63 hold rows 0-63 x columns
// [0, N/2), lanes 64-127 the same rows x columns [N/2, N) (the cta_group::2, M=128
// data-path layout) -- so no MMA work is spent on rows of the next segment.  For the
// gate-up GEMM the tail tile's B is staged as [gate 0-63 | up 0-63] (CTA 0) and
// [gate 64-127 | up 64-127] (CTA 1), so each lane still holds the gate and up
// values of its features and SwiGLU stays fused.  (FSEP_GEMM_MTAIL=0 / policy
// bit 12 falls back to the masked M=256 tile.)
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>

#include "kernels/grouped_gemm.cuh"
#include "kernels/sm100_ptx.cuh"

namespace fsep {

#ifdef FSEP_GEMM_STALLS
// Stall accounting (dev builds, -DFSEP_GEMM_STALLS): cycles each role spends in its
// barrier waits, summed over CTAs: [0] MMA waits for operands (full), [1] MMA waits
// for a free accumulator (tempty), [2] producer waits for a free stage (empty),
// [3] epilogue waits for an accumulator (tfull), [4] MMA-warp lifetime,
// [5] epilogue busy (drain) cycles, [6] producer readiness + wave-barrier waits.
__device__ unsigned long long g_gemm_stall[8];
#define FSEP_STALL_T0() const long long _t0 = clock64()
#define FSEP_STALL_ADD(acc) (acc) += clock64() - _t0
#else
#define FSEP_STALL_T0()
#define FSEP_STALL_ADD(acc)
#endif

namespace gemm2 {
constexpr int BM = 256, BN = 256, BK = 64, STAGES = 6;
constexpr int HALF = 128;                       // rows of A / columns of B per CTA
constexpr int A_BYTES = HALF * BK * 2;          // 16 KB
constexpr int B_BYTES = HALF * BK * 2;          // 16 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;  // per CTA
#ifndef FSEP_EPI_WARPS
#define FSEP_EPI_WARPS 8
#endif
constexpr int EPI_WARPS = FSEP_EPI_WARPS;  // 8: 4 TMEM lane quarters x 2 column halves; 4: quarters, both halves each
static_assert(EPI_WARPS == 8 || EPI_WARPS == 4, "epilogue warps must be 4 or 8");
constexpr int NHALF = EPI_WARPS == 8 ? 1 : 2;  // column halves per epilogue warp
constexpr int THREADS = 64 + EPI_WARPS * 32;
constexpr int MAX_GROUPS = 128;  // groups = hosted experts (<= kMaxExperts)
constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + 512;  // stages + barriers (tile tables are static smem)
// SwiGLU-bwd epilogue: per-warp [32 rows][32 fp32] transpose tile (XOR-swizzled float4 slots)
constexpr int EPI_STAGE_OFF = STAGES * STAGE_BYTES + 512;
constexpr int EPI_STAGE_BYTES = EPI_WARPS * 32 * 32 * 4;
// bf16 epilogues: per-warp [32 rows][64 B] row-piece transpose tile
constexpr int EPI_STAGE16_BYTES = EPI_WARPS * 32 * 64;
constexpr int smem_bytes(int epi) {
  return (epi == kEpiSwigluBwd || epi == kEpiBf16) ? 1024 + EPI_STAGE_OFF + EPI_STAGE_BYTES
                                                   : 1024 + EPI_STAGE_OFF + EPI_STAGE16_BYTES;
}
static_assert(1024 + EPI_STAGE_OFF + EPI_STAGE_BYTES + (2 * MAX_GROUPS + 1) * 4 <= 232448,
              "SwiGLU-bwd staging + tile tables exceed shared memory");

// Coalesced store of a warp's 32 row pieces of 64 B (32 bf16): lane r holds row
// r's piece in v[0..3]; the pieces are transposed through a 2 KB smem tile
// (XOR-swizzled 16-B slots, conflict-free both ways) so that every store
// instruction writes 8 rows x 64 contiguous bytes instead of 32 scattered 16-B
// pieces.  dst(rr) gives row rr's destination (nullptr: row not stored).
__device__ __forceinline__ void sts128(uint32_t a, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a) : "memory");
  return v;
}

// Coalesced store of a warp's 32 row pieces of 64 B (32 bf16): lane r holds row
// r's piece in v[0..3]; the pieces are transposed through a 2 KB smem tile
// (XOR-swizzled 16-B slots, conflict-free both ways) so that every store
// instruction writes 8 rows x 64 contiguous bytes instead of 32 scattered 16-B
// pieces.  dst(rr) gives row rr's destination (nullptr: row not stored).
template <typename Dst>
__device__ __forceinline__ void warp_store_rows64(uint32_t stg, const uint4 (&v)[4], Dst dst) {
  const int lane = static_cast<int>(threadIdx.x & 31);
#pragma unroll
  for (int q = 0; q < 4; ++q) sts128(stg + 16 * (lane * 4 + (q ^ ((lane >> 1) & 3))), v[q]);
  __syncwarp();
  const int sub = lane >> 2, cg = lane & 3;
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int rr = it * 8 + sub;
    const uint4 x = lds128(stg + 16 * (rr * 4 + (cg ^ ((rr >> 1) & 3))));
    auto* d = dst(rr);
    if (d != nullptr) reinterpret_cast<uint4*>(d)[cg] = x;
  }
  __syncwarp();
}

// Same for 128-B row pieces (64 bf16): 8 lanes per row, 4 rows per store
// instruction; nval = valid 16-B pieces of each row (columns past N are not stored).
template <typename Dst>
__device__ __forceinline__ void warp_store_rows128(uint32_t stg, const uint4 (&v)[8], int nval, Dst dst) {
  const int lane = static_cast<int>(threadIdx.x & 31);
#pragma unroll
  for (int q = 0; q < 8; ++q) sts128(stg + 16 * (lane * 8 + (q ^ (lane & 7))), v[q]);
  __syncwarp();
  const int sub = lane >> 3, cg = lane & 7;
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int rr = it * 4 + sub;
    const uint4 x = lds128(stg + 16 * (rr * 8 + (cg ^ (rr & 7))));
    auto* d = dst(rr);
    if (d != nullptr && cg < nval) reinterpret_cast<uint4*>(d)[cg] = x;
  }
  __syncwarp();
}

__device__ __forceinline__ void pack_row64(const float* v, uint4 (&o)[4]) {
  using ptx::pack_bf16;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    o[i] = make_uint4(pack_bf16(v[8 * i], v[8 * i + 1]), pack_bf16(v[8 * i + 2], v[8 * i + 3]),
                      pack_bf16(v[8 * i + 4], v[8 * i + 5]), pack_bf16(v[8 * i + 6], v[8 * i + 7]));
}
}  // namespace gemm2

template <bool kAMN, bool kBMN, bool kGroupK, int kEpi>
__global__ void __launch_bounds__(gemm2::THREADS, 1)
    grouped_gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                             const __grid_constant__ CUtensorMap tmB64, const GemmParams p) {
  using namespace gemm2;
  using namespace fsep::ptx;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);
  __shared__ int tile_start[MAX_GROUPS + 1];  // first tile of each group (static smem: LDS, not generic loads)
  // M-grouped: M tiles of each group.  K-grouped (every group has p.M / BM M tiles):
  // the group at each schedule position.
  __shared__ int group_mbs[MAX_GROUPS];
  int* group_id = group_mbs;

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int G = p.num_groups;
  const int nb = (p.N + BN - 1) / BN;
  const int cluster = blockIdx.x >> 1;
  const int nclusters = gridDim.x >> 1;

  // Schedule order of the groups.  K-grouped (wgrad): descending row count (ties:
  // lower index first), so that with the snake assignment below the tiles go out
  // longest-first -- the per-tile cost is the group's row count, which is very
  // skewed under Zipf routing (a static round robin left some CTA pairs with
  // ~20% more work than the mean).  M-grouped: identity (equal-cost tiles, and the
  // restored slots become ready in slot order).
  if (kGroupK) {
    for (int i = static_cast<int>(threadIdx.x); i < G; i += static_cast<int>(blockDim.x)) {
      int pos = i;
      if (!(p.policy & 0x200)) {
        const int ri = p.group_rows[i];
        pos = 0;
        for (int j = 0; j < G; ++j) {
          const int rj = p.group_rows[j];
          pos += (rj > ri || (rj == ri && j < i)) ? 1 : 0;
        }
      }
      group_id[pos] = i;
    }
    __syncthreads();
  }
  auto gid = [&](int gi) { return kGroupK ? group_id[gi] : gi; };
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int gi = 0; gi < G; ++gi) {
      tile_start[gi] = acc;
      acc += (kGroupK ? p.M / BM : (group_mbs[gi] = (p.group_rows[gi] + BM - 1) / BM)) * nb;
    }
    tile_start[G] = acc;
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);   // leader's arrive_expect_tx (+ both CTAs' tx bytes)
      mbar_init(&empty_bar[s], 1);  // MMA commit (multicast)
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);               // MMA commit (multicast)
      mbar_init(&tempty_bar[s], 2 * EPI_WARPS);  // both CTAs' epilogue warps (leader's copy is used)
    }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 1) tmem_alloc_pair<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total_tiles = tile_start[G];

  int gdec = 0;
  auto decode = [&](int t, int& g, int& mb, int& nbk) {
    // every role walks its tiles in increasing order: resume the group search
    while (tile_start[gdec + 1] <= t) ++gdec;
    g = gid(gdec);
    const int local = t - tile_start[gdec];
    const int mbs = kGroupK ? p.M / BM : group_mbs[gdec];
    raster_tile(local, mbs, nb, p.raster == 0 ? 16 : p.raster, kGroupK, mb, nbk);  // default: 16-tile m-chunks
  };
  auto k_blocks = [&](int g) { return kGroupK ? p.group_rows[g] / BK : p.K / BK; };
  // M=128 tail tile: the group's last 256-row tile holds only 128 (padded) rows.  The
  // gate-up GEMM needs the 64-row-box B map for its [gate|up] halves (policy bit 13).
  const bool tails_ok = !kGroupK && !(p.policy & 0x1000) &&
                        (kEpi != kEpiSwigluFwd || (p.policy & 0x2000));
  auto m_tail = [&](int g, int mb) { return tails_ok && p.group_rows[g] - mb * BM <= HALF; };
  // Tile of this CTA pair in wave w.  K-grouped: snake order (even waves ascending,
  // odd waves descending over the pairs), so consecutive waves hand the costlier
  // tiles of the descending-cost list to alternate ends -- LPT-like balance.
  // M-grouped: plain round robin (equal-cost tiles; the snake measured 4% slower
  // there).  Tile indices increase with w for every pair (the group search relies on it).
  auto wave_tile = [&](int w) {
    return w * nclusters + ((kGroupK && (w & 1) && !(p.policy & 0x200)) ? nclusters - 1 - cluster : cluster);
  };

  if (warp == 0) {
    // ------------------------------------------------------------ producer (both CTAs)
    if (elect_one()) {
      // default: both operands evict_last (measured best: concurrent tiles share both A and B panels)
      const uint64_t pol_a = pick_policy((p.policy & 3) ? (p.policy & 3) : 3, false);
      const uint64_t pol_b = pick_policy(((p.policy >> 2) & 3) ? ((p.policy >> 2) & 3) : 3, false);
      int s = 0;
      uint32_t ph = 0;
      int ready_g = -1;
      bool ready_live = true;
      bool wsync = p.wave_sync != nullptr;
      long long st_empty = 0, st_sync = 0;
      for (int w = 0, t = wave_tile(0); t < total_tiles; t = wave_tile(++w)) {
        {
          FSEP_STALL_T0();
          if (wsync && w > 0 && w <= kWaveSyncMax)  // CTAs with a tile in wave w
            wsync = wave_barrier(p.wave_sync + (w - 1), 2 * min(nclusters, total_tiles - w * nclusters));
          FSEP_STALL_ADD(st_sync);
        }
        int g, mb, nbk;
        decode(t, g, mb, nbk);
        const int nk = k_blocks(g);
        const int row0 = p.group_off[g];
        if (!kGroupK && g != ready_g && ready_live) {
          FSEP_STALL_T0();
          ready_live = wait_group_ready(p, g);  // false: timed out (error raised), stop waiting
          ready_g = g;
          FSEP_STALL_ADD(st_sync);
        }
        const bool mt = m_tail(g, mb);
        // this CTA's first A row (M-grouped: within the group); a tail tile stages 64 rows per CTA
        // (the 128-row box also brings the next 64 rows, which the M=128 MMA does not read)
        const int m_half = mb * BM + rank * (mt ? HALF / 2 : HALF);
        // this CTA's first B column; a last N tile with <= 128 live columns runs as
        // UMMA N=128, each CTA providing 64 columns
        const bool n_tail = p.N - nbk * BN <= HALF && !(p.policy & 0x100);
        const int n_half = nbk * BN + rank * (n_tail ? HALF / 2 : HALF);
        // policy bit 14: odd waves stream K backwards, so they start on the k-blocks of the
        // panels the previous wave touched last (still in L2).  Only the load order changes:
        // the MMA accumulates in arrival order.
        const bool krev = (p.policy & 0x4000) && (w & 1);
        for (int kq = 0; kq < nk; ++kq) {
          const int kb = krev ? nk - 1 - kq : kq;
          {
            FSEP_STALL_T0();
            mbar_wait(&empty_bar[s], ph ^ 1);
            FSEP_STALL_ADD(st_empty);
          }
          uint8_t* sA = smem + s * STAGE_BYTES;
          uint8_t* sB = sA + A_BYTES;
          if (leader) mbar_arrive_expect_tx(&full_bar[s], 2 * STAGE_BYTES);
          if (!kAMN) {
            tma_load_2d_pair(sA, &tmA, &full_bar[s], kb * BK, row0 + m_half, pol_a);
          } else {
#pragma unroll
            for (int i = 0; i < HALF / 64; ++i)
              tma_load_2d_pair(sA + i * 8192, &tmA, &full_bar[s], m_half + i * 64, row0 + kb * BK, pol_a);
          }
          if (!kGroupK) {
            if (kEpi == kEpiSwigluFwd && mt) {  // [gate 64 | up 64] of this CTA's feature half
              const int f0 = nbk * BN + rank * (HALF / 2);
              tma_load_3d_pair(sB, &tmB64, &full_bar[s], kb * BK, f0, g, pol_b);
              tma_load_3d_pair(sB + B_BYTES / 2, &tmB64, &full_bar[s], kb * BK, f0 + HALF, g, pol_b);
            } else if (!kBMN) {
              tma_load_3d_pair(sB, &tmB, &full_bar[s], kb * BK, n_half, g, pol_b);
            } else {
#pragma unroll
              for (int i = 0; i < HALF / 64; ++i)
                tma_load_3d_pair(sB + i * 8192, &tmB, &full_bar[s], n_half + i * 64, kb * BK, g, pol_b);
            }
          } else {
#pragma unroll
            for (int i = 0; i < HALF / 64; ++i)
              tma_load_2d_pair(sB + i * 8192, &tmB, &full_bar[s], n_half + i * 64, row0 + kb * BK, pol_b);
          }
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
#ifdef FSEP_GEMM_STALLS
      atomicAdd(&g_gemm_stall[2], static_cast<unsigned long long>(st_empty));
      atomicAdd(&g_gemm_stall[6], static_cast<unsigned long long>(st_sync));
#endif
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader CTA)
    if (leader) {
      constexpr uint32_t idesc = ptx::idesc_bf16(BM, BN, kAMN, kBMN);
      constexpr uint32_t idesc_tail = ptx::idesc_bf16(BM, BN / 2, kAMN, kBMN);  // last N tile with <= 128 columns
      constexpr uint32_t idesc_m = ptx::idesc_bf16(HALF, BN, kAMN, kBMN);          // M=128 tail tile
      constexpr uint32_t idesc_m_tail = ptx::idesc_bf16(HALF, BN / 2, kAMN, kBMN);  // M=128 and N=128
      int s = 0;
      uint32_t ph = 0;
      int it = 0;
      long long st_full = 0, st_tempty = 0;
#ifdef FSEP_GEMM_STALLS
      const long long t_begin = clock64();
#endif
      for (int w = 0, t = wave_tile(0); t < total_tiles; t = wave_tile(++w), ++it) {
        int g, mb, nbk;
        decode(t, g, mb, nbk);
        const int nk = k_blocks(g);
        const int as = it & 1;
        const uint32_t aph = (it >> 1) & 1;
        {
          FSEP_STALL_T0();
          mbar_wait(&tempty_bar[as], aph ^ 1);
          FSEP_STALL_ADD(st_tempty);
        }
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + as * BN;
        const bool ntl = p.N - nbk * BN <= HALF && !(p.policy & 0x100);
        const uint32_t id = m_tail(g, mb) ? (ntl ? idesc_m_tail : idesc_m) : (ntl ? idesc_tail : idesc);
        for (int kb = 0; kb < nk; ++kb) {
          {
            FSEP_STALL_T0();
            mbar_wait(&full_bar[s], ph);
            FSEP_STALL_ADD(st_full);
          }
          tc_fence_after();
          if (lane == 0) {
            const uint32_t a0 = smem_u32(smem + s * STAGE_BYTES);
            const uint32_t b0 = a0 + A_BYTES;
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              const uint64_t ad = kAMN ? smem_desc(a0 + k * 2048, 8192, 1024) : smem_desc(a0 + k * 32, 16, 1024);
              const uint64_t bd = kBMN ? smem_desc(b0 + k * 2048, 8192, 1024) : smem_desc(b0 + k * 32, 16, 1024);
              umma_bf16_pair(tmem_d, ad, bd, id, (kb | k) ? 1u : 0u);
            }
            umma_commit_pair(&empty_bar[s], 0x3);
          }
          __syncwarp();
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        // accumulator ready (for an empty K range this arrives at once: nothing pending)
        if (lane == 0) umma_commit_pair(&tfull_bar[as], 0x3);
        __syncwarp();
      }
#ifdef FSEP_GEMM_STALLS
      if (lane == 0) {
        atomicAdd(&g_gemm_stall[0], static_cast<unsigned long long>(st_full));
        atomicAdd(&g_gemm_stall[1], static_cast<unsigned long long>(st_tempty));
        atomicAdd(&g_gemm_stall[4], static_cast<unsigned long long>(clock64() - t_begin));
      }
#endif
    }
  } else {
    // ------------------------------------------------------------ epilogue (both CTAs)
    const uint32_t quarter = warp & 3;
    const int half0 = NHALF == 1 ? static_cast<int>(warp - 2) >> 2 : 0;
    const int r = static_cast<int>(quarter * 32 + lane);  // row within this CTA's 128 rows
    int it = 0;
    long long st_tfull = 0, st_drain = 0;
    for (int w = 0, t = wave_tile(0); t < total_tiles; t = wave_tile(++w), ++it) {
      int g, mb, nbk;
      decode(t, g, mb, nbk);
      const int as = it & 1;
      const uint32_t aph = (it >> 1) & 1;
      const int m_half = mb * BM + static_cast<int>(rank) * HALF;
      // Tail tile (M=128 MMA): this CTA holds tile rows rank*64 + [0, 64); TMEM lanes 64-127
      // repeat those rows for the upper half of the columns (see the file comment).
      const bool mt = m_tail(g, mb);
      const int tn = (p.N - nbk * BN <= HALF && !(p.policy & 0x100)) ? HALF : BN;  // MMA N of this tile
      // first tile row of this warp's 32 lanes; TMEM columns [tc0, tc0 + tcw) of this warp;
      // logical column of TMEM column tc = lc0 + (tc - tc0)
      const int wrow0 = mt ? mb * BM + static_cast<int>(rank) * (HALF / 2) + static_cast<int>(quarter & 1) * 32
                           : m_half + static_cast<int>(quarter) * 32;
      const int tcw = mt ? tn / 4 : HALF;
      const bool valid = kGroupK || mt || m_half < p.group_rows[g];
      if (kEpi == kEpiSwigluBwd && valid && !mt && !(p.policy & 0x8000)) {
        // While the MMAs of this tile run, pull this row's h slice (one 128-feature
        // block: 256 contiguous bf16 = 512 B) into L2 so the epilogue loads hit L2.
        for (int half = half0; half < half0 + NHALF; ++half) {
          const int f0 = nbk * BN + half * 128;
          if (f0 < p.N) {
            const __nv_bfloat16* hrow = static_cast<const __nv_bfloat16*>(p.aux) +
                                        (static_cast<long long>(p.group_off[g]) + m_half + r) * p.ld_aux + (f0 / 128) * 256;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], 512;" ::"l"(hrow) : "memory");
          }
        }
      }
      {
        FSEP_STALL_T0();
        mbar_wait(&tfull_bar[as], aph);
        FSEP_STALL_ADD(st_tfull);
      }
#ifdef FSEP_GEMM_STALLS
      const long long t_drain = clock64();
#endif
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((quarter * 32) << 16) + as * BN;
      if (valid)
#pragma unroll 1
      for (int half = half0; half < half0 + NHALF; ++half) {
        const int tc0 = half * tcw;                                                 // TMEM columns of this half
        const int lc0 = mt ? static_cast<int>(quarter >> 1) * (tn / 2) + tc0 : tc0;  // their logical columns
        if (kEpi == kEpiF32) {
          // fp32 rows, stored coalesced: each 32-column chunk goes out as two 64-B row
          // pieces through the per-warp transpose tile (8 rows x 64 B per store)
          const bool empty_k = k_blocks(g) == 0;
          const uint32_t stg = ptx::smem_u32(smem + EPI_STAGE_OFF) + (warp - 2) * 2048;
          float* ob = static_cast<float*>(p.out) + static_cast<long long>(g) * p.out_group_stride +
                      static_cast<long long>(m_half + quarter * 32) * p.ldo;
#pragma unroll 1
          for (int j = 0; j < 4; ++j) {
            const int c = half * 128 + j * 32;
            const int col = nbk * BN + c;
            if (col >= p.N) break;
            float v[32];
            if (empty_k) {
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = 0.f;
            } else {
              tmem_ld32(taddr + c, v);
            }
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              uint4 o[4];
#pragma unroll
              for (int q = 0; q < 4; ++q)
                o[q] = make_uint4(__float_as_uint(v[16 * hh + 4 * q]), __float_as_uint(v[16 * hh + 4 * q + 1]),
                                  __float_as_uint(v[16 * hh + 4 * q + 2]), __float_as_uint(v[16 * hh + 4 * q + 3]));
              warp_store_rows64(stg, o, [&](int rr) { return ob + rr * p.ldo + col + 16 * hh; });
            }
          }
        } else if (kEpi == kEpiBf16) {
          const long long row = p.group_off[g] + wrow0 + static_cast<int>(lane);
          __nv_bfloat16* out = bf16_out_row(p, row);  // own row (row scatter resolved per lane)
#ifndef FSEP_EPI_ROW64
          // 64-column passes, 128-B row pieces (fewer, larger remote writes for the row scatter)
          const uint32_t stg = ptx::smem_u32(smem + EPI_STAGE_OFF) + (warp - 2) * 4096;
#pragma unroll 1
          for (int j = 0; j * 64 < tcw; ++j) {
            const int tc = tc0 + j * 64;                 // TMEM column
            const int col = nbk * BN + lc0 + j * 64;     // logical output column
            if (col >= p.N) break;
            const int w = min(64, tcw - j * 64);         // 64, or 32 for an M=128 x N=128 tail tile
            float v[64];
            tmem_ld32(taddr + tc, *reinterpret_cast<float(*)[32]>(v));
            if (w > 32 && col + 32 < p.N) tmem_ld32(taddr + tc + 32, *reinterpret_cast<float(*)[32]>(v + 32));
            uint4 o[8];
            pack_row64(v, *reinterpret_cast<uint4(*)[4]>(o));
            pack_row64(v + 32, *reinterpret_cast<uint4(*)[4]>(o + 4));
            warp_store_rows128(stg, o, min(w / 8, (p.N - col) / 8), [&](int rr) {
              __nv_bfloat16* d = reinterpret_cast<__nv_bfloat16*>(
                  __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(out), rr));
              return d == nullptr ? d : d + col;
            });
          }
#else
          const uint32_t stg = ptx::smem_u32(smem + EPI_STAGE_OFF) + (warp - 2) * 2048;
#pragma unroll 1
          for (int j = 0; j * 32 < tcw; ++j) {
            const int col = nbk * BN + lc0 + j * 32;
            if (col >= p.N) break;
            float v[32];
            tmem_ld32(taddr + tc0 + j * 32, v);
            uint4 o[4];
            pack_row64(v, o);
            warp_store_rows64(stg, o, [&](int rr) {
              __nv_bfloat16* d = reinterpret_cast<__nv_bfloat16*>(
                  __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(out), rr));
              return d == nullptr ? d : d + col;
            });
          }
#endif
        } else if (kEpi == kEpiSwigluFwd) {
          // tile columns [0,128) = gate f0.., [128,256) = up f0..; this warp: f in [64*half, 64*half+64)
          const uint32_t stg = ptx::smem_u32(smem + EPI_STAGE_OFF) + (warp - 2) * 2048;
          const long long row0 = p.group_off[g] + wrow0;
          __nv_bfloat16* hb = static_cast<__nv_bfloat16*>(p.out) + nbk * BN;
          __nv_bfloat16* ab = static_cast<__nv_bfloat16*>(p.out2) + nbk * (BN / 2);
          // full tile: TMEM columns [0,128) gate, [128,256) up of the 128 features; this warp's
          // features half*64 + [0,64).  Tail tile: TMEM [0,64) gate, [64,128) up of the features
          // (quarter>>1)*64 + [0,64) (the [gate|up] B staging); this warp's 32 of them.
          const int nf = mt ? 1 : 2;
#pragma unroll 1
          for (int j = 0; j < nf; ++j) {
            const int tg = mt ? half * 32 : half * 64 + j * 32;                      // TMEM column of the gates
            const int tu = tg + (mt ? 64 : 128);                                    // ... of the ups
            const int f = mt ? static_cast<int>(quarter >> 1) * 64 + half * 32 : tg;  // feature within the block
            float gv[32], uv[32];
            tmem_ld32(taddr + tg, gv);
            tmem_ld32(taddr + tu, uv);
            uint4 o[4];
            pack_row64(gv, o);
            warp_store_rows64(stg, o, [&](int rr) { return hb + (row0 + rr) * p.ldo + f; });
            pack_row64(uv, o);
            warp_store_rows64(stg, o, [&](int rr) { return hb + (row0 + rr) * p.ldo + 128 + f; });
#pragma unroll
            for (int q = 0; q < 32; ++q) gv[q] = silu_f(gv[q]) * uv[q];
            pack_row64(gv, o);
            warp_store_rows64(stg, o, [&](int rr) { return ab + (row0 + rr) * p.ldo2 + f; });
          }
        } else {  // kEpiSwigluBwd
          // dAct arrives one row per lane (TMEM 32x32b); it is transposed through a
          // per-warp smem tile so that the h loads and dH stores are row-contiguous
          // across lanes (4 lanes x 16 B of one row, 8 rows per instruction) rather
          // than one 16-B piece of 32 different rows per instruction.  The h loads
          // of chunk j+1 are in flight while chunk j computes.
          const uint32_t stg = ptx::smem_u32(smem + EPI_STAGE_OFF) + (warp - 2) * 4096;
          const long long row0 = p.group_off[g] + wrow0;
          const int sub = static_cast<int>(lane >> 2), cg = static_cast<int>(lane & 3);
          const __nv_bfloat16* hb = static_cast<const __nv_bfloat16*>(p.aux);
          __nv_bfloat16* db = static_cast<__nv_bfloat16*>(p.out);
          int nch = 0;
          for (int j = 0; j * 32 < tcw; ++j)
            if (nbk * BN + lc0 + j * 32 < p.N) nch = j + 1;
          auto hcol = [&](int j) {
            const int f = nbk * BN + lc0 + j * 32;
            return static_cast<long long>((f / 128) * 256 + (f % 128) + cg * 8);
          };
          auto load_h = [&](int j, uint4 (&gq)[4], uint4 (&uq)[4]) {
            const long long hc = hcol(j);
#pragma unroll
            for (int it = 0; it < 4; ++it) {
              const __nv_bfloat16* hr = hb + (row0 + it * 8 + sub) * p.ld_aux + hc;
              gq[it] = *reinterpret_cast<const uint4*>(hr);
              uq[it] = *reinterpret_cast<const uint4*>(hr + 128);
            }
          };
          uint4 gq[4], uq[4];
          if (nch > 0) load_h(0, gq, uq);
#pragma unroll 1
          for (int j = 0; j < nch; ++j) {
            float da[32];
            tmem_ld32(taddr + tc0 + j * 32, da);
#pragma unroll
            for (int q = 0; q < 8; ++q)
              sts128(stg + 16 * (lane * 8 + (q ^ (lane & 7))),
                     make_uint4(__float_as_uint(da[4 * q]), __float_as_uint(da[4 * q + 1]),
                                __float_as_uint(da[4 * q + 2]), __float_as_uint(da[4 * q + 3])));
            uint4 gn[4], un[4];
            if (j + 1 < nch) load_h(j + 1, gn, un);
            __syncwarp();
            const long long hc = hcol(j);
#pragma unroll
            for (int it = 0; it < 4; ++it) {
              const int rr = it * 8 + sub;
              const uint4 d0 = lds128(stg + 16 * (rr * 8 + ((2 * cg) ^ (rr & 7))));
              const uint4 d1 = lds128(stg + 16 * (rr * 8 + ((2 * cg + 1) ^ (rr & 7))));
              const float d[8] = {__uint_as_float(d0.x), __uint_as_float(d0.y), __uint_as_float(d0.z),
                                  __uint_as_float(d0.w), __uint_as_float(d1.x), __uint_as_float(d1.y),
                                  __uint_as_float(d1.z), __uint_as_float(d1.w)};
              const __nv_bfloat16* gb = reinterpret_cast<const __nv_bfloat16*>(&gq[it]);
              const __nv_bfloat16* ub = reinterpret_cast<const __nv_bfloat16*>(&uq[it]);
              float dg[8], du[8];
#pragma unroll
              for (int q = 0; q < 8; ++q) {
                const float gg = __bfloat162float(gb[q]);
                const float uu = __bfloat162float(ub[q]);
                const float sg = sigmoid_f(gg);
                du[q] = d[q] * gg * sg;
                dg[q] = d[q] * uu * sg * (1.0f + gg * (1.0f - sg));
              }
              __nv_bfloat16* dr = db + (row0 + rr) * p.ldo + hc;
              *reinterpret_cast<uint4*>(dr) = make_uint4(pack_bf16(dg[0], dg[1]), pack_bf16(dg[2], dg[3]),
                                                         pack_bf16(dg[4], dg[5]), pack_bf16(dg[6], dg[7]));
              *reinterpret_cast<uint4*>(dr + 128) = make_uint4(pack_bf16(du[0], du[1]), pack_bf16(du[2], du[3]),
                                                               pack_bf16(du[4], du[5]), pack_bf16(du[6], du[7]));
            }
            __syncwarp();
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              gq[i] = gn[i];
              uq[i] = un[i];
            }
          }
        }
      }
#ifdef FSEP_GEMM_STALLS
      st_drain += clock64() - t_drain;
#endif
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (p.policy & 0x400)
          mbar_arrive_cluster(&tempty_bar[as], 0);  // FSEP_TMEM_RELEASE=cluster (A/B)
        else
          mbar_arrive_remote(&tempty_bar[as], 0);
      }
    }
#ifdef FSEP_GEMM_STALLS
    if (lane == 0) {
      atomicAdd(&g_gemm_stall[3], static_cast<unsigned long long>(st_tfull));
      atomicAdd(&g_gemm_stall[5], static_cast<unsigned long long>(st_drain));
    }
#endif
  }
  __syncthreads();
  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_pair<512>(tmem_base);
  }
}

}  // namespace fsep
